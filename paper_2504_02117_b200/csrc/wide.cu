// wide.cu -- a3 / a5 for WIDE strided operands: the block-GMRES multi-Gram
// [V_0 .. V_j]^T W and multi-update W -= [V_0 .. V_j] H over the row-major basis
// (N x (m+1)k, ld = (m+1)k).  A tile of T rows of a strided
// operand is T separate row segments: one producer thread moves it with 2-D TMA
// tensor-map copies (cp.async.bulk.tensor.2d, boxes of <= 256 columns x T rows,
// out-of-range rows zero-filled by the TMA unit) into a 2-stage ring.  (A
// lane-parallel cp.async staging was measured ~5x slower: ~30 instructions per
// row in the producer warps.)  The consumers run on the FP64 tensor cores (DMMA):
//   gram  : each warp owns a set of 8-column blocks of V (all rows of the tile),
//           per-CTA partials in global memory, a second kernel sums them in a
//           fixed order (deterministic);
//   update: warps = (row block) x (K quarter); the K-quarter partials are summed
//           in a fixed order through shared memory, plus a W.
#include <cuda.h>

#include "bk_internal.h"
#include "ptx.cuh"

namespace bk {
namespace {

constexpr int WNC = 512;         // consumer threads (16 warps)
constexpr int WNW = WNC / 32;
constexpr int WSTAGES = 4;

// One operand: rows [r0, r0 + nr) x cols [0, w) of a row-major array with ld,
// staged densely by TMA ([T][bw] panels; out-of-range rows / columns zero-filled).
struct Opnd {
    const double* p;
    int64_t ld;
    int w, wp;       // columns, staged row width (even; = nbox * bw for V)
    int off;         // byte offset inside a stage
    int nbox, bw;    // TMA boxes per tile row: nbox boxes of bw columns (panels [T][bw])
    int ps;          // panel stride in doubles (128-byte aligned TMA destinations)
};

struct WideArgs {
    int64_t n;
    int T, ntiles;
    int ns;          // ring stages (<= WSTAGES)
    int rb;          // update: row blocks of 8 per tile (T = 8 rb); warps = rb x (16 / rb) K slices
    int stage_bytes;
    Opnd V;          // n x ka
    Opnd W;          // n x kb (gram: Y operand; update: Xin, present iff a != 0)
    int ka, kb;
    bool hasW;
    // gram
    double* part;    // [gridDim.x * rs][ka * kb]
    int rs;          // row slices: with fewer column blocks than warps, warp = (block, slice)
    // update
    double a, s;
    const double* H; // ka x k row-major
    int hfrag;       // s H staged as B fragments in shared memory
    double* out;
    int64_t ldo;
    const int* halt;
};

__device__ __forceinline__ void wide_setup(uint64_t* full, uint64_t* empty) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < WSTAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], WNW);
        }
        mbar_fence_init();
    }
}

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// producer (one thread): the tile's V boxes (panels [T][bw]) and the W box
__device__ __forceinline__ void wide_produce(const WideArgs& w, const CUtensorMap* tmV, const CUtensorMap* tmW,
                                             unsigned char* smem, uint64_t* full, uint64_t* empty) {
    if ((threadIdx.x & 31) != 0) return;
    const uint32_t vbytes = (uint32_t)w.V.nbox * w.T * w.V.bw * 8u;
    // W contiguous (ld == width == staged width): one 1-D bulk copy per tile (a 2-D box of
    // narrow rows costs one TMA row request per row); the ragged last tile by hand
    const bool w1d = w.hasW && w.W.ld == w.W.w && w.W.wp == w.W.w && (((uintptr_t)w.W.p) & 15) == 0;
    const uint64_t pol = evict_first_policy();
    int i = 0;
    for (int tile = blockIdx.x; tile < w.ntiles; tile += gridDim.x, ++i) {
        const int s = i % w.ns;
        if (i >= w.ns) mbar_wait(&empty[s], ((i / w.ns) - 1) & 1);
        unsigned char* st = smem + s * w.stage_bytes;
        const int r0 = tile * w.T;
        const int nr = (int)((w.n - r0) < w.T ? (w.n - r0) : w.T);
        uint32_t wbytes = 0;
        bool wbulk = false;
        if (w.hasW) {
            if (w1d && nr == w.T && ((uint32_t)nr * w.W.w * 8u) % 16u == 0u) {
                wbulk = true;
                wbytes = (uint32_t)nr * w.W.w * 8u;
            } else if (w1d) {   // last tile: plain copy + zero rows (visible through the arrive below)
                double* d = reinterpret_cast<double*>(st + w.W.off);
                for (int e = 0; e < w.T * w.W.w; ++e) d[e] = e < nr * w.W.w ? w.W.p[(int64_t)r0 * w.W.w + e] : 0.0;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before any later bulk copy here
            } else {
                wbytes = (uint32_t)w.T * w.W.wp * 8u;
            }
        }
        mbar_expect_tx(&full[s], vbytes + wbytes);
        for (int p = 0; p < w.V.nbox; ++p)
            tma2d(st + w.V.off + p * w.V.ps * 8, tmV, p * w.V.bw, r0, &full[s]);
        if (wbulk) bulk_g2s(st + w.W.off, w.W.p + (int64_t)r0 * w.W.w, wbytes, &full[s], pol);
        else if (w.hasW && !w1d) tma2d(st + w.W.off, tmW, 0, r0, &full[s]);
    }
}

// ------------------------------------------------------------------ wide Gram: G = V^T W
// NAW: column blocks of V per warp (block i = warp + 16 t); NBK = ceil(kb / 8)
template <int NAW, int NBK>
__global__ void __launch_bounds__(WNC + 32, 1)
gram_wide_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmW, const WideArgs w) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + w.ns * w.stage_bytes);
    uint64_t* empty = full + WSTAGES;
    wide_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == WNW) {
        wide_produce(w, &tmV, &tmW, smem, full, empty);
        return;
    }
    const int kq = lane & 3, mg = lane >> 2;
    const int NA = (w.ka + 7) / 8;
    // rs > 1 (NAW == 1, NA * rs <= 16): warp owns block warp % NA and rows slice warp / NA
    const int RS = w.rs;
    const int wb = RS > 1 ? warp % NA : warp, sl = RS > 1 ? warp / NA : 0;
    const bool wact = sl < RS;
    double acc[NAW][NBK][2];
#pragma unroll
    for (int t = 0; t < NAW; ++t)
#pragma unroll
        for (int j = 0; j < NBK; ++j) acc[t][j][0] = acc[t][j][1] = 0.0;
    const int wpW = w.W.wp, bw = w.V.bw;
    // per owned block: offset of this lane's column in the stage (panel, column), or -1
    int voff[NAW];
#pragma unroll
    for (int t = 0; t < NAW; ++t) {
        const int c = 8 * (wb + WNW * t) + mg;
        voff[t] = c < w.ka ? (c / bw) * w.V.ps + (c % bw) : -1;
    }
    int woff[NBK];
#pragma unroll
    for (int j = 0; j < NBK; ++j) woff[j] = (8 * j + mg) < w.kb ? 8 * j + mg : -1;
    int i = 0;
    for (int tile = blockIdx.x; tile < w.ntiles; tile += gridDim.x, ++i) {
        const int s = i % w.ns;
        mbar_wait(&full[s], (i / w.ns) & 1);
        const unsigned char* st = smem + s * w.stage_bytes;
        const double* Vs = reinterpret_cast<const double*>(st + w.V.off);
        const double* Ws = reinterpret_cast<const double*>(st + w.W.off);
        for (int q0 = 4 * sl; wact && q0 < w.T; q0 += 4 * RS) {
            const int r = q0 + kq;
            double b[NBK];
#pragma unroll
            for (int j = 0; j < NBK; ++j) b[j] = woff[j] >= 0 ? Ws[r * wpW + woff[j]] : 0.0;
#pragma unroll
            for (int t = 0; t < NAW; ++t) {
                if (wb + WNW * t < NA) {   // warp-uniform
                    const double av = voff[t] >= 0 ? Vs[voff[t] + r * bw] : 0.0;
#pragma unroll
                    for (int j = 0; j < NBK; ++j) dmma(acc[t][j][0], acc[t][j][1], av, b[j]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    // this CTA's (row slice's) partial: block (blk, j): rows 8 blk + mg, cols 8 j + 2 kq (+1)
    if (!wact) return;
    double* P = w.part + ((int64_t)blockIdx.x * RS + sl) * w.ka * w.kb;
#pragma unroll
    for (int t = 0; t < NAW; ++t) {
        const int blk = wb + WNW * t;
        if (blk >= NA) continue;
        const int a = 8 * blk + mg;
#pragma unroll
        for (int j = 0; j < NBK; ++j) {
            const int b = 8 * j + 2 * kq;
            if (a < w.ka && b < w.kb) P[a * w.kb + b] = acc[t][j][0];
            if (a < w.ka && b + 1 < w.kb) P[a * w.kb + b + 1] = acc[t][j][1];
        }
    }
}

// G[e] = sum_{c < nblk} part[c][e], fixed order
__global__ void wide_reduce_kernel(const double* __restrict__ part, int nblk, int nout, double* __restrict__ G) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nout; e += gridDim.x * blockDim.x) {
        double v[8];
        double s = 0.0;
        int c = 0;
        for (; c + 8 <= nblk; c += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + (int64_t)(c + u) * nout + e);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; c < nblk; ++c) s += __ldcg(part + (int64_t)c * nout + e);
        G[e] = s;
    }
}

// ------------------------------------------------------------------ wide update: out = a W + s V H
// T = 8 rb rows per tile (rb = 16, 8, 4 row blocks); warp = (row block warp % rb, K slice warp / rb of 16 / rb);
// NK = ceil(k / 8) output column blocks.  H (ka x k) B fragments read through L1 (__ldg).
template <int NK>
__global__ void __launch_bounds__(WNC + 32, 1)
upd_wide_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmW, const WideArgs w) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + w.ns * w.stage_bytes);
    uint64_t* empty = full + WSTAGES;
    double* red = reinterpret_cast<double*>(smem + w.ns * w.stage_bytes + 64);   // [16/rb][8 rb][8 NK]
    double* sHf = red + 4 * 32 * 8 * NK;   // s H as m8n8k4 B fragments [ks][j][lane] (if it fits)
    if (w.halt && *w.halt) return;
    wide_setup(full, empty);
    const int NQ = (w.ka + 3) / 4;                 // K steps of 4
    if (w.hfrag) {
        for (int e = threadIdx.x; e < NQ * NK * 32; e += blockDim.x) {
            const int l = e & 31, j = (e >> 5) % NK, ks = (e >> 5) / NK;
            const int c = 4 * ks + (l & 3), oc = 8 * j + (l >> 2);
            sHf[e] = (c < w.ka && oc < w.kb) ? w.s * w.H[(int64_t)c * w.kb + oc] : 0.0;
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == WNW) {
        wide_produce(w, &tmV, &tmW, smem, full, empty);
        return;
    }
    const int kq = lane & 3, mg = lane >> 2;
    const int RB = w.rb, QS = WNW / RB;
    const int rb4 = warp % RB, q4 = warp / RB;
    const int qs = (NQ * q4) / QS, qe = (NQ * (q4 + 1)) / QS;
    const int k = w.kb, KP8 = 8 * NK;
    const int wpW = w.W.wp, bw = w.V.bw;
    int i = 0;
    for (int tile = blockIdx.x; tile < w.ntiles; tile += gridDim.x, ++i) {
        const int s = i % w.ns;
        mbar_wait(&full[s], (i / w.ns) & 1);
        const unsigned char* st = smem + s * w.stage_bytes;
        const double* Vs = reinterpret_cast<const double*>(st + w.V.off);
        const double* Ws = reinterpret_cast<const double*>(st + w.W.off);
        const int64_t r0 = (int64_t)tile * w.T;
        const int nr = (int)((w.n - r0) < w.T ? (w.n - r0) : w.T);
        double d[NK][2];
#pragma unroll
        for (int j = 0; j < NK; ++j) d[j][0] = d[j][1] = 0.0;
        const int row = 8 * rb4 + mg;   // < T
        {
            int c = 4 * qs + kq;
            int pnl = c / bw, cc = c - pnl * bw;          // (panel, column) tracked incrementally
            const double* hp = w.H + (int64_t)c * k;
            for (int ks = qs; ks < qe; ++ks) {
                const double av = c < w.ka ? Vs[pnl * w.V.ps + row * bw + cc] : 0.0;
#pragma unroll
                for (int j = 0; j < NK; ++j) {
                    double bv;
                    if (w.hfrag) {
                        bv = sHf[(ks * NK + j) * 32 + lane];
                    } else {
                        const int oc = 8 * j + mg;
                        bv = (c < w.ka && oc < k) ? w.s * __ldg(hp + oc) : 0.0;
                    }
                    dmma(d[j][0], d[j][1], av, bv);
                }
                c += 4;
                hp += 4 * k;
                cc += 4;
                if (cc >= bw) { cc -= bw; ++pnl; }
            }
        }
        // K-slice partials -> shared memory, fixed-order sum (+ a W) by all consumers
        const int TT = 8 * RB;
#pragma unroll
        for (int j = 0; j < NK; ++j) {
            double* rp = red + ((q4 * TT + row) * KP8 + 8 * j + 2 * kq);
            rp[0] = d[j][0];
            rp[1] = d[j][1];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(WNC));
        for (int e = threadIdx.x; e < TT * k; e += WNC) {
            const int r = e / k, cc = e - r * k;
            double v = red[r * KP8 + cc];
            for (int q = 1; q < QS; ++q) v += red[(q * TT + r) * KP8 + cc];
            if (w.hasW) v = fma(w.a, Ws[r * wpW + cc], v);
            if (r < nr) w.out[(r0 + r) * w.ldo + cc] = v;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(WNC));
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 2-D fp64 tensor map over rows [0, n) x cols [0, w) of a row-major array (ld), box bw x T
bool encode(CUtensorMap* m, const double* p, int64_t n, int w, int64_t ld, int bw, int T) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || ((uintptr_t)p & 15) || (ld * 8) % 16 || bw > 256 || T > 256 || (bw * 8) % 16) return false;
    cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
    cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)T};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool geometry(WideArgs& w, int64_t n, int T, CUtensorMap* tmV, CUtensorMap* tmW) {
    auto r128 = [](int x) { return (x + 127) & ~127; };
    w.V.nbox = (w.V.w + 255) / 256;
    w.V.bw = ((w.V.w + w.V.nbox - 1) / w.V.nbox + 1) & ~1;
    w.V.wp = w.V.nbox * w.V.bw;
    w.V.ps = r128(T * w.V.bw * 8) / 8;
    w.W.wp = (w.W.w + 1) & ~1;
    w.T = T;
    w.V.off = 0;
    w.W.off = w.V.nbox * w.V.ps * 8;
    w.stage_bytes = r128(w.W.off + (w.hasW ? T * w.W.wp * 8 : 0));
    w.n = n;
    const int64_t nt = (n + T - 1) / T;
    if (nt * T >= (1ll << 31)) return false;
    w.ntiles = (int)nt;
    if (!encode(tmV, w.V.p, n, w.V.w, w.V.ld, w.V.bw, T)) return false;
    if (w.hasW) {
        if (!encode(tmW, w.W.p, n, w.W.w, w.W.ld, w.W.wp, T)) return false;
    } else {
        *tmW = *tmV;
    }
    return true;
}

void set_smem_attr(const void* fn) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); }

}  // namespace

bool wide_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("BK_WIDE");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

static int wide_row_slices(int ka) {
    const int NA = (ka + 7) / 8;
    return NA < WNW ? WNW / NA : 1;
}
size_t gram_wide_ws_doubles(int ka, int kb, int num_sms) {
    return (size_t)num_sms * wide_row_slices(ka) * ka * kb + 64;
}

// G (ka x kb) = V^T W, V: n x ka (ldv), W: n x kb (ldw); false = not applicable
bool launch_gram_wide(int64_t n, int ka, int kb, const double* V, int64_t ldv, const double* W, int64_t ldw,
                      double* G, double* part, int num_sms, cudaStream_t st) {
    if (!wide_enabled() || n <= 0 || ka < 16 || ka > 16 * 8 * 16 || kb < 1 || kb > 32) return false;
    WideArgs w{};
    w.V = Opnd{V, ldv, ka, 0, 0, 0, 0};
    w.W = Opnd{W, ldw, kb, 0, 0, 0, 0};
    w.hasW = true;
    w.ka = ka;
    w.kb = kb;
    w.part = part;
    // tile rows: V and W tiles of <= ~100 KB per stage, multiple of 4
    int T = (48 * 1024) / ((ka + 8) * 8 + ((kb + 1) & ~1) * 8);
    T = T > 256 ? 256 : (T & ~3);
    if (T < 4) return false;
    CUtensorMap tmV, tmW;
    if (!geometry(w, n, T, &tmV, &tmW)) return false;
    w.ns = WSTAGES;
    while (w.ns > 2 && w.ns * w.stage_bytes + 64 > 227 * 1024) --w.ns;
    const int smem = w.ns * w.stage_bytes + 64;
    if (smem > 227 * 1024) return false;
    const int NA = (ka + 7) / 8, NBK = (kb + 7) / 8;
    const int naw = (NA + WNW - 1) / WNW;
    const int grid = w.ntiles < num_sms ? w.ntiles : num_sms;
    w.rs = wide_row_slices(ka);   // idle warps take row slices of the tile
    bool ok = false;
#define BK_GW(A, B)                                                                           \
    if (!ok && naw <= A && NBK == B) {                                                        \
        static bool at = false;                                                               \
        if (!at) { set_smem_attr((const void*)gram_wide_kernel<A, B>); at = true; }           \
        BK_KERNEL(gram_wide_kernel<A, B><<<grid, WNC + 32, smem, st>>>(tmV, tmW, w));          \
        ok = true;                                                                            \
    }
    BK_GW(1, 1) BK_GW(1, 2) BK_GW(1, 3) BK_GW(1, 4) BK_GW(2, 1) BK_GW(2, 2) BK_GW(2, 3) BK_GW(2, 4)
    BK_GW(4, 1) BK_GW(4, 2) BK_GW(4, 3) BK_GW(4, 4) BK_GW(8, 1) BK_GW(8, 2) BK_GW(8, 3)
#undef BK_GW
    if (!ok) return false;
    const int nout = ka * kb;
    BK_KERNEL(wide_reduce_kernel<<<(nout + 255) / 256 < 2 * num_sms ? (nout + 255) / 256 : 2 * num_sms, 256, 0, st>>>(
        part, grid * w.rs, nout, G));
    return true;
}

// out = a Xin + s V H (Xin, out: n x k, ld k; V: n x ka, ldv; H: ka x k device); false = not applicable.
// dry: plan only (a column split launches its parts only after every part has a plan, so a
// false return never leaves a partial update behind for the caller's fallback)
static bool update_wide_impl(const UpdArgs& u, cudaStream_t st, bool dry) {
    // (small systems: launch-bound, the generic kernel has less fixed cost for narrow V)
    const bool small_n = u.n < 65536;
    if (!wide_enabled() || u.n <= 0 || u.kp < (small_n ? 16 : 4) || u.kp > 2048 || u.k < 1 || u.k > 32 || u.W)
        return false;
    if (!u.P || !u.C || u.ldo < u.k) return false;
    if ((const double*)u.out == u.P) return false;
    if (u.a != 0.0 && !u.Xin) return false;
    WideArgs w{};
    w.V = Opnd{u.P, u.ldp, u.kp, 0, 0, 0, 0};
    w.W = Opnd{u.a != 0.0 ? u.Xin : nullptr, u.ldxin, u.k, 0, 0, 0, 0};
    w.hasW = u.a != 0.0;
    w.ka = u.kp;
    w.kb = u.k;
    w.a = u.a;
    w.s = u.s;
    w.H = u.C;
    w.out = u.out;
    w.ldo = u.ldo;
    w.halt = u.halt;
    CUtensorMap tmV, tmW;
    const int NK = (u.k + 7) / 8;
    const int red_bytes = 128 * 8 * NK * 8;
    const int64_t hf_bytes = (int64_t)((u.kp + 3) / 4) * NK * 32 * 8;
    // s H as shared-memory B fragments, then the largest tile (128, 64 or 32 rows) with >= 2
    // stages: a tile costs two CTA barriers and a single producer thread ~1 us per tile (16 / 8-row
    // tiles measured slower than the generic kernel); without the fragments every DMMA waits on
    // an L1 load of H (c3 GMRES(64), k = 12: 64-row tiles without them 1.3 TB/s, 32-row tiles
    // with them 3.4-3.8 TB/s), so a wider V is split instead
    int smem = 0;
    bool ok = false;
    if (hf_bytes <= 64 * 1024) {
        for (int rb = small_n ? 4 : 16; rb >= 4 && !ok; rb /= 2) {
            // (the TMA encoder refuses some large boxes, e.g. 240 columns x 128 rows: next tile size)
            if (!geometry(w, u.n, 8 * rb, &tmV, &tmW)) continue;
            w.rb = rb;
            for (int ns = WSTAGES; ns >= 2 && !ok; --ns) {
                const int64_t need = (int64_t)ns * w.stage_bytes + 64 + red_bytes + hf_bytes;
                if (need <= 227 * 1024) {
                    w.ns = ns;
                    w.hfrag = 1;
                    smem = (int)need;
                    ok = true;
                }
            }
        }
    }
    if (!ok) {
        // too wide for a 32-row tile with its H fragments: split the contraction over V's columns,
        // out = a Xin + s V[:, :h] H[:h, :], then out += s V[:, h:] H[h:, :] (the second part reads
        // out as its Xin, tile by tile before writing it: one extra N x k round trip per split)
        if (u.kp < 32 || ((uintptr_t)u.out & 15) || (u.ldo * 8) % 16) return false;   // out must be a TMA operand
        const int h = ((u.kp / 2) + 3) & ~3;
        UpdArgs lo = u, hi = u;
        lo.kp = h;
        hi.P = u.P + h;
        hi.C = u.C + (int64_t)h * u.k;
        hi.kp = u.kp - h;
        hi.a = 1.0;
        hi.Xin = u.out;
        hi.ldxin = u.ldo;
        return update_wide_impl(lo, st, dry) && update_wide_impl(hi, st, dry);
    }
    if (dry) return true;
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = w.ntiles < nsm ? w.ntiles : nsm;
#define BK_UW(K)                                                                              \
    if (NK == K) {                                                                            \
        static bool at = false;                                                               \
        if (!at) { set_smem_attr((const void*)upd_wide_kernel<K>); at = true; }               \
        BK_KERNEL(upd_wide_kernel<K><<<grid, WNC + 32, smem, st>>>(tmV, tmW, w));              \
        return true;                                                                          \
    }
    BK_UW(1) BK_UW(2) BK_UW(3) BK_UW(4)
#undef BK_UW
    return false;
}

bool launch_update_wide(const UpdArgs& u, cudaStream_t st) {
    return update_wide_impl(u, st, true) && update_wide_impl(u, st, false);
}

}  // namespace bk
