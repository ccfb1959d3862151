// gram_mma.cu -- a3 block Gram G = X^T Y on the FP64 tensor cores (DMMA).
//
// PAPER.md §1: the k x k block inner products through which the columns
// of a block Krylov method exchange information.  On B200 the Gram at
// k >= 8 is a genuine dense contraction over N rows (AI = ka kb / (4 (ka+kb))
// FLOP/byte, 2-4 at k = 16-32), so it runs on the tensor cores: tcgen05 has
// no FP64 kind, the FP64 tensor path is mma.sync.m8n8k4.f64 (SASS DMMA).
//  * grid = chunks x panels (panel = 32 columns of X for multi-Grams);
//  * each warp walks 4-row quads of its CTA's contiguous row chunk; one quad
//    is one k-step of m8n8k4: A = X^T (8 x 4), B = Y (4 x 8), C = G block;
//    fragments are loaded straight from global memory (each instruction reads
//    64 contiguous bytes of 4 rows), 4 quads in flight per warp;
//  * the 8 warps' accumulators are combined in shared memory in fixed order,
//    the CTA partial is written, and the LAST CTA to finish (atomic ticket)
//    sums all partials in fixed order -> one launch, bitwise reproducible.
#include "bk_internal.h"

namespace bk {
namespace {

constexpr int kWarps = 8;
constexpr int kQuadUnroll = 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// NA x NB blocks of 8 x 8 per panel: KAP = 8 NA columns of X, KBP = 8 NB columns of Y
template <int NA, int NB>
__global__ void __launch_bounds__(kWarps * 32)
gram_mma_kernel(int64_t n, int ka, int kb, const double* __restrict__ X, int64_t ldx,
                const double* __restrict__ Y, int64_t ldy, double* __restrict__ part, int* __restrict__ ticket,
                double* __restrict__ G, int npanels, int64_t rows_per_chunk) {
    constexpr int KAP = 8 * NA, KBP = 8 * NB, NOUT = KAP * KBP;
    extern __shared__ double s_red[];            // kWarps * NOUT
    __shared__ int s_last;
    const int panel = blockIdx.x % npanels;
    const int64_t chunk = blockIdx.x / npanels;
    const int nchunks = gridDim.x / npanels;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kq = lane & 3, mg = lane >> 2;      // k index (row in quad), m/n group
    const int pa = panel * KAP;
    const int64_t r0 = chunk * rows_per_chunk;
    const int64_t r1 = (n < r0 + rows_per_chunk) ? n : r0 + rows_per_chunk;

    double acc[NA][NB][2];
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    bool am[NA], bm[NB];
#pragma unroll
    for (int i = 0; i < NA; ++i) am[i] = pa + 8 * i + mg < ka;
#pragma unroll
    for (int j = 0; j < NB; ++j) bm[j] = 8 * j + mg < kb;
    const double* xb = X + pa + mg;
    const double* yb = Y + mg;

    // quads of this warp: rows r0 + 4 (warp + kWarps q) + kq
    for (int64_t base = r0 + 4 * warp; base < r1; base += (int64_t)4 * kWarps * kQuadUnroll) {
        double av[kQuadUnroll][NA], bv[kQuadUnroll][NB];
#pragma unroll
        for (int u = 0; u < kQuadUnroll; ++u) {
            const int64_t row = base + (int64_t)4 * kWarps * u + kq;
            const bool rin = row < r1;
#pragma unroll
            for (int i = 0; i < NA; ++i) av[u][i] = (rin && am[i]) ? __ldg(xb + row * ldx + 8 * i) : 0.0;
#pragma unroll
            for (int j = 0; j < NB; ++j) bv[u][j] = (rin && bm[j]) ? __ldg(yb + row * ldy + 8 * j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kQuadUnroll; ++u)
#pragma unroll
            for (int i = 0; i < NA; ++i)
#pragma unroll
                for (int j = 0; j < NB; ++j) dmma(acc[i][j][0], acc[i][j][1], av[u][i], bv[u][j]);
    }
    // C fragment: lane holds G[8i + mg][8j + 2 kq + {0,1}]
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            double* d = s_red + warp * NOUT + (8 * i + mg) * KBP + 8 * j + 2 * kq;
            d[0] = acc[i][j][0];
            d[1] = acc[i][j][1];
        }
    __syncthreads();
    double* out = part + ((int64_t)chunk * npanels + panel) * NOUT;
    for (int o = tid; o < NOUT; o += kWarps * 32) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += s_red[w * NOUT + o];
        out[o] = s;
    }
    // last CTA reduces all partials in fixed order
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(ticket, 1) == (int)gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int o = warp; o < ka * kb; o += kWarps) {
        const int a = o / kb, b = o % kb;
        const int pnl = a / KAP, ai = a % KAP;
        const int idx = ai * KBP + b;
        double s = 0.0;
        for (int c = lane; c < nchunks; c += 32) s += __ldcg(part + ((int64_t)c * npanels + pnl) * NOUT + idx);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        if (lane == 0) G[(int64_t)a * kb + b] = s;
    }
    if (tid == 0) *ticket = 0;
}

int chunks_for(int64_t n, int npanels, int num_sms) {
    // ~2 CTAs per SM in total, at least ~512 rows per chunk
    int64_t want = (n + 511) / 512;
    int64_t cap = (2 * (int64_t)num_sms + npanels - 1) / npanels;
    if (cap < 1) cap = 1;
    int64_t c = want < cap ? want : cap;
    return (int)(c < 1 ? 1 : c);
}

template <int NA, int NB>
void gram_mma_t(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* G,
                double* part, int* ticket, int num_sms, cudaStream_t st) {
    constexpr int KAP = 8 * NA;
    const int npanels = (ka + KAP - 1) / KAP;
    const int nchunks = chunks_for(n, npanels, num_sms);
    const int64_t rpc = ((n + nchunks - 1) / nchunks + 3) & ~(int64_t)3;
    const size_t smem = (size_t)kWarps * 64 * NA * NB * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gram_mma_kernel<NA, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    BK_KERNEL(gram_mma_kernel<NA, NB><<<nchunks * npanels, kWarps * 32, smem, st>>>(
        n, ka, kb, X, ldx, Y, ldy, part, ticket, G, npanels, rpc > 0 ? rpc : 4));
}

template <int NA>
void gram_mma_a(int nb, int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                double* G, double* part, int* ticket, int num_sms, cudaStream_t st) {
    switch (nb) {
        case 1: return gram_mma_t<NA, 1>(n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
        case 2: return gram_mma_t<NA, 2>(n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
        case 3: return gram_mma_t<NA, 3>(n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
        default: return gram_mma_t<NA, 4>(n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
    }
}

}  // namespace

size_t gram_mma_ws_doubles(int64_t n, int ka, int kb, int num_sms) {
    const int na = ka >= 32 ? 4 : (ka + 7) / 8;
    const int nb = (kb + 7) / 8;
    const int npanels = (ka + 8 * na - 1) / (8 * na);
    return (size_t)chunks_for(n, npanels, num_sms) * npanels * 64 * na * nb;
}

void launch_gram_mma(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                     double* G, double* part, int* ticket, int num_sms, cudaStream_t st) {
    const int na = ka >= 32 ? 4 : (ka + 7) / 8;
    const int nb = (kb + 7) / 8;
    switch (na) {
        case 1: return gram_mma_a<1>(nb, n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
        case 2: return gram_mma_a<2>(nb, n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
        case 3: return gram_mma_a<3>(nb, n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
        default: return gram_mma_a<4>(nb, n, ka, kb, X, ldx, Y, ldy, G, part, ticket, num_sms, st);
    }
}

}  // namespace bk
