// blas.cu -- a3 block Gram, a5 block update and the small N x k helpers (sm_100a).
//
// a3  G = X^T Y  (§1: k x k block inner products through which
//     the columns exchange information).  Deterministic two-stage reduction:
//     stage 1: each CTA reduces a contiguous row chunk into register tiles
//     (TA x TB outputs per thread, R row-groups per CTA), combines its groups
//     in shared memory in fixed order and writes one partial; stage 2: one warp
//     per output sums the partials in fixed order (strided lanes + fixed
//     shuffle tree).  Same bits on every run; no atomics.
// a5  out = a X + s P C (+ w W)  (block axpy of the Krylov recurrences).  A
//     group of LANES threads owns one row, C is staged in shared memory and
//     the P row is broadcast with warp shuffles, so P, X and out are each
//     streamed once.
#include "bk_internal.h"

namespace bk {
namespace {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ gram
template <int KAP, int KBP>
struct GramCfg {
    static constexpr int TA = KAP < 4 ? KAP : 4;
    static constexpr int TB = KBP < 4 ? KBP : 4;
    static constexpr int NA = KAP / TA, NB = KBP / TB;
    static constexpr int G = NA * NB;          // threads per row-group
    static constexpr int R = kThreads / G;     // row-groups per CTA
};

// partials layout: [chunk][panel][KAP*KBP]
template <int KAP, int KBP>
__global__ void __launch_bounds__(kThreads)
gram_partial_kernel(int64_t n, int ka, int kb, const double* __restrict__ X, int64_t ldx,
                    const double* __restrict__ Y, int64_t ldy, double* __restrict__ part,
                    int npanels, int64_t rows_per_chunk) {
    using Cfg = GramCfg<KAP, KBP>;
    constexpr int TA = Cfg::TA, TB = Cfg::TB, G = Cfg::G, R = Cfg::R, NB = Cfg::NB;
    __shared__ double s_red[R * KAP * KBP > 1 ? R * KAP * KBP : 1];
    const int panel = blockIdx.x % npanels;
    const int64_t chunk = blockIdx.x / npanels;
    const int tid = threadIdx.x, g = tid / G, j = tid % G;
    const int a0 = (j / NB) * TA, b0 = (j % NB) * TB;
    const int pa = panel * KAP;                 // panel column offset into X
    const int64_t r0 = chunk * rows_per_chunk;
    const int64_t r1 = (n < r0 + rows_per_chunk ? n : r0 + rows_per_chunk);
    double acc[TA][TB];
#pragma unroll
    for (int u = 0; u < TA; ++u)
#pragma unroll
        for (int v = 0; v < TB; ++v) acc[u][v] = 0.0;
    bool amask[TA], bmask[TB];
#pragma unroll
    for (int u = 0; u < TA; ++u) amask[u] = pa + a0 + u < ka;
#pragma unroll
    for (int v = 0; v < TB; ++v) bmask[v] = b0 + v < kb;
    const double* xb = X + pa + a0;
    const double* yb = Y + b0;
    int64_t i = r0 + g;
    for (; i + R < r1; i += 2 * R) {            // 2 rows in flight per thread
        double x0[TA], y0[TB], x1[TA], y1[TB];
#pragma unroll
        for (int u = 0; u < TA; ++u) x0[u] = amask[u] ? __ldg(xb + i * ldx + u) : 0.0;
#pragma unroll
        for (int v = 0; v < TB; ++v) y0[v] = bmask[v] ? __ldg(yb + i * ldy + v) : 0.0;
#pragma unroll
        for (int u = 0; u < TA; ++u) x1[u] = amask[u] ? __ldg(xb + (i + R) * ldx + u) : 0.0;
#pragma unroll
        for (int v = 0; v < TB; ++v) y1[v] = bmask[v] ? __ldg(yb + (i + R) * ldy + v) : 0.0;
#pragma unroll
        for (int u = 0; u < TA; ++u)
#pragma unroll
            for (int v = 0; v < TB; ++v) acc[u][v] = fma(x0[u], y0[v], acc[u][v]);
#pragma unroll
        for (int u = 0; u < TA; ++u)
#pragma unroll
            for (int v = 0; v < TB; ++v) acc[u][v] = fma(x1[u], y1[v], acc[u][v]);
    }
    for (; i < r1; i += R) {
        double x0[TA], y0[TB];
#pragma unroll
        for (int u = 0; u < TA; ++u) x0[u] = amask[u] ? __ldg(xb + i * ldx + u) : 0.0;
#pragma unroll
        for (int v = 0; v < TB; ++v) y0[v] = bmask[v] ? __ldg(yb + i * ldy + v) : 0.0;
#pragma unroll
        for (int u = 0; u < TA; ++u)
#pragma unroll
            for (int v = 0; v < TB; ++v) acc[u][v] = fma(x0[u], y0[v], acc[u][v]);
    }
    // fixed-order combination of the R row-groups
#pragma unroll
    for (int u = 0; u < TA; ++u)
#pragma unroll
        for (int v = 0; v < TB; ++v) s_red[g * KAP * KBP + (a0 + u) * KBP + (b0 + v)] = acc[u][v];
    __syncthreads();
    double* out = part + ((int64_t)chunk * npanels + panel) * (KAP * KBP);
    for (int o = tid; o < KAP * KBP; o += kThreads) {
        double s = 0.0;
        for (int r = 0; r < R; ++r) s += s_red[r * KAP * KBP + o];
        out[o] = s;
    }
}

// one warp per output: lanes sum chunks strided by 32 in order, then a fixed
// xor-shuffle tree.  Writes G row-major ka x kb.
template <int KAP, int KBP>
__global__ void gram_reduce_kernel(const double* __restrict__ part, int nchunks, int npanels,
                                   int ka, int kb, double* __restrict__ G) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= ka * kb) return;
    const int a = warp / kb, b = warp % kb;
    const int panel = a / KAP, ai = a % KAP;
    const int o = ai * KBP + b;
    double s = 0.0;
    for (int c = lane; c < nchunks; c += 32) s += part[((int64_t)c * npanels + panel) * (KAP * KBP) + o];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if (lane == 0) G[(int64_t)a * kb + b] = s;
}

int nchunks_for(int64_t n, int npanels, int num_sms) {
    int64_t want = (n + 1023) / 1024;                       // >= ~1024 rows per chunk
    int64_t cap = (int64_t)4 * num_sms / (npanels > 4 ? 4 : npanels);
    if (cap < num_sms) cap = num_sms;
    int64_t c = want < cap ? want : cap;
    return (int)(c < 1 ? 1 : c);
}

int pow2_at_least(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

template <int KAP, int KBP>
void gram_t(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
            double* G, double* part, int num_sms, cudaStream_t st) {
    const int npanels = (ka + KAP - 1) / KAP;
    const int nchunks = nchunks_for(n, npanels, num_sms);
    const int64_t rpc = (n + nchunks - 1) / nchunks;
    BK_KERNEL(gram_partial_kernel<KAP, KBP><<<nchunks * npanels, kThreads, 0, st>>>(n, ka, kb, X, ldx, Y, ldy, part,
                                                                       npanels, rpc > 0 ? rpc : 1));
    const int warps = ka * kb;
    BK_KERNEL(gram_reduce_kernel<KAP, KBP><<<(warps * 32 + 255) / 256, 256, 0, st>>>(part, nchunks, npanels, ka, kb, G));
}

template <int KAP>
void gram_a(int kbp, int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y,
            int64_t ldy, double* G, double* part, int num_sms, cudaStream_t st) {
    switch (kbp) {
        case 1: return gram_t<KAP, 1>(n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 2: return gram_t<KAP, 2>(n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 4: return gram_t<KAP, 4>(n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 8: return gram_t<KAP, 8>(n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 16: return gram_t<KAP, 16>(n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        default: return gram_t<KAP, 32>(n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
    }
}

// ------------------------------------------------------------------ column dots
template <int KP>
__global__ void __launch_bounds__(kThreads)
coldot_partial_kernel(int64_t n, int k, const double* __restrict__ X, int64_t ldx,
                      const double* __restrict__ Y, int64_t ldy, const double* __restrict__ Y2,
                      int64_t ldy2, double* __restrict__ part, int64_t rows_per_chunk) {
    constexpr int R = kThreads / KP;
    __shared__ double s1[kThreads], s2[kThreads];
    const int tid = threadIdx.x, g = tid / KP, c = tid % KP;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_chunk;
    const int64_t r1 = (n < r0 + rows_per_chunk ? n : r0 + rows_per_chunk);
    double d1 = 0.0, d2 = 0.0;
    if (c < k) {
        for (int64_t i = r0 + g; i < r1; i += R) {
            const double x = __ldg(X + i * ldx + c);
            d1 = fma(x, __ldg(Y + i * ldy + c), d1);
            if (Y2) d2 = fma(x, __ldg(Y2 + i * ldy2 + c), d2);
        }
    }
    s1[tid] = d1; s2[tid] = d2;
    __syncthreads();
    if (tid < KP) {
        double a = 0.0, b = 0.0;
        for (int r = 0; r < R; ++r) { a += s1[r * KP + tid]; b += s2[r * KP + tid]; }
        part[(int64_t)blockIdx.x * 2 * KP + tid] = a;
        part[(int64_t)blockIdx.x * 2 * KP + KP + tid] = b;
    }
}

template <int KP>
__global__ void coldot_reduce_kernel(const double* __restrict__ part, int nchunks, int k, double* d,
                                     double* d2) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int o = warp; o < 2 * k; o += blockDim.x >> 5) {
        const int which = o / k, c = o % k;
        if (which == 1 && d2 == nullptr) continue;
        double s = 0.0;
        for (int ch = lane; ch < nchunks; ch += 32) s += part[(int64_t)ch * 2 * KP + which * KP + c];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        if (lane == 0) (which ? d2 : d)[c] = s;
    }
}

template <int KP>
void coldot_t(int64_t n, int k, const double* X, int64_t ldx, const double* Y, int64_t ldy,
              const double* Y2, int64_t ldy2, double* d, double* d2, double* part, int num_sms,
              cudaStream_t st) {
    const int nchunks = nchunks_for(n, 1, num_sms);
    const int64_t rpc = (n + nchunks - 1) / nchunks;
    BK_KERNEL(coldot_partial_kernel<KP><<<nchunks, kThreads, 0, st>>>(n, k, X, ldx, Y, ldy, Y2, ldy2, part,
                                                           rpc > 0 ? rpc : 1));
    BK_KERNEL(coldot_reduce_kernel<KP><<<1, 1024, 0, st>>>(part, nchunks, k, d, d2));
}

// ------------------------------------------------------------------ update
// One group of LANES = KP threads per row, lane l owns output column l.  All
// PASSES rows of a thread issue their X / W / P loads before any arithmetic
// (many independent 8-byte loads in flight per thread, coalesced across the
// group); the P row is then broadcast with warp shuffles against C rows held
// in shared memory.  kp > KP (GMRES multi-update) loops over KP-wide chunks.
constexpr int kUpdPasses = 8;

template <int KP>
__global__ void __launch_bounds__(kThreads)
update_kernel(const UpdArgs a) {
    constexpr int LANES = KP;
    constexpr int RPP = kThreads / LANES;
    constexpr int PASSES = kUpdPasses;
    __shared__ double s_C[KP * KP];
    if (a.halt && *a.halt) return;
    const int tid = threadIdx.x, grp = tid / LANES, lane = tid % LANES;
    const int k = a.k, kp = a.kp;
    const bool lane_in = lane < k;
    const int64_t base = (int64_t)blockIdx.x * (RPP * PASSES) + grp;
    double xv[PASSES], wv[PASSES], acc[PASSES];
#pragma unroll
    for (int q = 0; q < PASSES; ++q) {
        const int64_t row = base + (int64_t)q * RPP;
        const bool act = row < a.n && lane_in;
        xv[q] = (act && a.a != 0.0) ? a.Xin[row * a.ldxin + lane] : 0.0;
        wv[q] = (act && a.W) ? a.W[row * a.ldw + lane] : 0.0;
        acc[q] = 0.0;
    }
    for (int cb = 0; cb < kp; cb += KP) {
        const int nc = min(KP, kp - cb);
        if (cb > 0) __syncthreads();
        for (int i = tid; i < KP * KP; i += kThreads) {
            const int r = i / KP, c = i % KP;
            s_C[i] = (r < nc && c < k) ? a.C[(int64_t)(cb + r) * k + c] : 0.0;
        }
        double pv[PASSES];
#pragma unroll
        for (int q = 0; q < PASSES; ++q) {
            const int64_t row = base + (int64_t)q * RPP;
            pv[q] = (row < a.n && lane < nc) ? a.P[row * a.ldp + cb + lane] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int qq = 0; qq < KP; ++qq) {
            if (qq < nc) {                                   // CTA-uniform
                const double cv = s_C[qq * KP + lane];
#pragma unroll
                for (int q = 0; q < PASSES; ++q) {
                    const double p = (LANES == 1) ? pv[q] : __shfl_sync(0xffffffffu, pv[q], qq, LANES);
                    acc[q] = fma(p, cv, acc[q]);
                }
            }
        }
    }
    const double w = a.W ? (a.w_dev ? a.w_host * *a.w_dev : a.w_host) : 0.0;
#pragma unroll
    for (int q = 0; q < PASSES; ++q) {
        const int64_t row = base + (int64_t)q * RPP;
        if (row < a.n && lane_in) {
            double v = a.s * acc[q];
            v = fma(a.a, xv[q], v);
            v = fma(w, wv[q], v);
            a.out[row * a.ldo + lane] = v;
        }
    }
}

template <int KP>
void update_k(const UpdArgs& a, cudaStream_t st) {
    constexpr int RPP = kThreads / KP;
    const unsigned grid = (unsigned)((a.n + RPP * kUpdPasses - 1) / (RPP * kUpdPasses));
    if (grid) BK_KERNEL(update_kernel<KP><<<grid, kThreads, 0, st>>>(a));
}

// ------------------------------------------------------------------ misc
__global__ void row_scale_kernel(int64_t n, int k, const double* __restrict__ dinv,
                                 const double* __restrict__ X, int64_t ldx, double* __restrict__ out,
                                 int64_t ldo) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * k) return;
    const int64_t i = t / k;
    const int c = (int)(t % k);
    out[i * ldo + c] = dinv[i] * X[i * ldx + c];
}

__global__ void diag_inv_kernel(int64_t n, int64_t row_offset, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ col, const double* __restrict__ val,
                                double* __restrict__ dinv) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
        if ((int64_t)col[p] == i + row_offset) d += val[p];
    dinv[i] = d != 0.0 ? 1.0 / d : 1.0;
}

// NEXT-4 Chebyshev step (oracle O9): first step (AZ == null): W = cr D^-1 R, Z = W;
// else W = cw W + cr D^-1 (R - AZ), Z += W.  Rows in groups of k threads (coalesced
// row-major), grid-stride over row blocks.  W, AZ: ld = k.
__global__ void cheb_step_kernel(int64_t n, int k, const double* __restrict__ R, int64_t ldr,
                                 const double* __restrict__ AZ, const double* __restrict__ dinv,
                                 double* __restrict__ W, double* __restrict__ Z, int64_t ldz, double cw, double cr) {
    const int rpb = blockDim.x / k;
    const int lr = threadIdx.x / k, c = threadIdx.x % k;
    if (lr >= rpb) return;
    for (int64_t i = (int64_t)blockIdx.x * rpb + lr; i < n; i += (int64_t)gridDim.x * rpb) {
        const double di = dinv[i];
        const double r = R[i * ldr + c];
        if (AZ == nullptr) {
            const double w = cr * (di * r);
            W[i * k + c] = w;
            Z[i * ldz + c] = w;
        } else {
            const double w = fma(cw, W[i * k + c], cr * (di * (r - AZ[i * k + c])));
            W[i * k + c] = w;
            Z[i * ldz + c] += w;
        }
    }
}

// Gershgorin bound of D^-1 A: max_i |dinv_i| sum_j |a_ij| (non-negative doubles order as
// their bit patterns: atomicMax on the bits is exact and order independent)
__global__ void gershgorin_kernel(int64_t n, const int32_t* __restrict__ rp, const double* __restrict__ val,
                                  const double* __restrict__ dinv, unsigned long long* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double g = 0.0;
    if (i < n) {
        double s = 0.0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) s += fabs(val[p]);
        g = s * fabs(dinv[i]);
    }
    for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(g));
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void pack_rows_kernel(int64_t nrows, int k, const int32_t* __restrict__ rows,
                                 const double* __restrict__ X, int64_t ldx, double* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nrows * k) return;
    const int64_t r = t / k;
    const int c = (int)(t % k);
    out[t] = X[(int64_t)rows[r] * ldx + c];
}

}  // namespace

size_t gram_ws_doubles(int64_t n, int ka, int kb, int num_sms) {
    const int kap = ka >= 32 ? 32 : pow2_at_least(ka);
    const int kbp = pow2_at_least(kb);
    const int npanels = (ka + kap - 1) / kap;
    return (size_t)nchunks_for(n, npanels, num_sms) * npanels * kap * kbp;
}

void launch_gram(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                 double* G, double* part, int num_sms, cudaStream_t st) {
    const int kap = ka >= 32 ? 32 : pow2_at_least(ka);
    const int kbp = pow2_at_least(kb);
    switch (kap) {
        case 1: return gram_a<1>(kbp, n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 2: return gram_a<2>(kbp, n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 4: return gram_a<4>(kbp, n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 8: return gram_a<8>(kbp, n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        case 16: return gram_a<16>(kbp, n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
        default: return gram_a<32>(kbp, n, ka, kb, X, ldx, Y, ldy, G, part, num_sms, st);
    }
}

size_t coldot_ws_doubles(int64_t n, int k, int num_sms) {
    return (size_t)nchunks_for(n, 1, num_sms) * 2 * 32;
}

void launch_coldot(int64_t n, int k, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                   const double* Y2, int64_t ldy2, double* d, double* d2, double* part, int num_sms,
                   cudaStream_t st) {
    const int kp = pow2_at_least(k);
    switch (kp) {
        case 1: return coldot_t<1>(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, part, num_sms, st);
        case 2: return coldot_t<2>(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, part, num_sms, st);
        case 4: return coldot_t<4>(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, part, num_sms, st);
        case 8: return coldot_t<8>(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, part, num_sms, st);
        case 16: return coldot_t<16>(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, part, num_sms, st);
        default: return coldot_t<32>(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, part, num_sms, st);
    }
}

bool use_stream_kernels() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("BK_STREAM");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

void launch_update(const UpdArgs& a, cudaStream_t st) {
    if (a.n <= 0) return;
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    if (launch_update_flat(a, nsm, st)) return;   // k, kp <= 4 (flat.cu)
    if (use_stream_kernels() && launch_update_stream(a, nsm, st)) return;
    // strided or wide P (GMRES basis): cp.async-staged DMMA multi-update
    if (a.kp >= 4 && !a.W && (a.kp > 32 || a.ldp != a.kp || a.ldo != a.k) && launch_update_wide(a, st)) return;
    const int kp = pow2_at_least(a.k);
    switch (kp) {
        case 1: return update_k<1>(a, st);
        case 2: return update_k<2>(a, st);
        case 4: return update_k<4>(a, st);
        case 8: return update_k<8>(a, st);
        case 16: return update_k<16>(a, st);
        default: return update_k<32>(a, st);
    }
}

void launch_row_scale(int64_t n, int k, const double* dinv, const double* X, int64_t ldx, double* out,
                      int64_t ldo, cudaStream_t st) {
    const int64_t t = n * k;
    if (t > 0) BK_KERNEL(row_scale_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(n, k, dinv, X, ldx, out, ldo));
}

void launch_extract_diag_inv(int64_t n, int64_t row_offset, const int32_t* rp, const int32_t* col,
                             const double* val, double* dinv, cudaStream_t st) {
    if (n > 0) BK_KERNEL(diag_inv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, row_offset, rp, col, val, dinv));
}

void launch_cheb_step(int64_t n, int k, const double* R, int64_t ldr, const double* AZ, const double* dinv,
                      double* W, double* Z, int64_t ldz, double cw, double cr, cudaStream_t st) {
    if (n <= 0) return;
    const int rpb = 256 / k;
    int64_t grid = (n + rpb - 1) / rpb;
    if (grid > 148 * 16) grid = 148 * 16;
    BK_KERNEL(cheb_step_kernel<<<(unsigned)grid, 256, 0, st>>>(n, k, R, ldr, AZ, dinv, W, Z, ldz, cw, cr));
}

void launch_gershgorin(int64_t n, const int32_t* rp, const double* val, const double* dinv, unsigned long long* out,
                       cudaStream_t st) {
    if (n > 0) BK_KERNEL(gershgorin_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, rp, val, dinv, out));
}

void launch_fill(double* p, int64_t n, double v, cudaStream_t st) {
    if (n > 0) BK_KERNEL(fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, n, v));
}

void launch_pack_rows(int64_t nrows, int k, const int32_t* rows, const double* X, int64_t ldx,
                      double* out, cudaStream_t st) {
    const int64_t t = nrows * k;
    if (t > 0) BK_KERNEL(pack_rows_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(nrows, k, rows, X, ldx, out));
}

}  // namespace bk
