// spmm.cu -- a1: block operator apply  Y = alpha (A X) C + beta Y  on sm_100a.
//
// PAPER.md §3: the BOP kernel "Y <- A X" loads the matrix once for
// all k columns.  B200 mapping:
//  * persistent, warp-specialised CTAs (3 per SM): one PRODUCER warp streams
//    CSR tiles (TR = 256 rows: row pointers, column ids, values -- one
//    contiguous range each) from HBM into a 2-stage shared-memory ring with
//    TMA bulk copies (cp.async.bulk + mbarrier complete_tx, evict-first L2
//    policy), so the matrix is read exactly once and several tiles are always
//    in flight; eight CONSUMER warps compute tile t while t+1 lands;
//  * a group of LANES = KP/VEC consumer threads owns one row; lane l holds
//    columns [l*VEC, l*VEC+VEC) (VEC = 4 -> one 256-bit gather of X per
//    nonzero); a row's gathers are issued in batches (B*VEC = 16 doubles)
//    before any FMA (memory-level parallelism for the L2-resident stencil
//    neighbours);
//  * Y is written once with streaming (evict-first) stores;
//  * the optional k x k_out coupling C is applied in the epilogue
//    (FP64 tensor cores for k >= 8), so the coupled apply costs no extra HBM pass.
// Band-structured matrices (stencils) take the windowed kernel (X band segments
// staged by TMA); row lists (boundary rows of a partitioned matrix) use a
// direct, unstaged kernel.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "bk_internal.h"
#include "dense_dev.cuh"
#include "ptx.cuh"
#include "reduce.cuh"

namespace bk {
namespace {

constexpr int kThreads = 256;    // consumer threads
constexpr int kTileRows = 256;   // rows per CSR tile
// X gathers in flight per row and thread: B rows of X (VEC doubles each), B*VEC = 16
template <int VEC>
struct Batch { static constexpr int B = VEC >= 8 ? 2 : (VEC >= 4 ? 4 : 8); };

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ void ld_x(const double* p, double (&x)[1]) { x[0] = __ldg(p); }
// VEC % 4 == 0: 256-bit loads (sm_100 LDG.E.ENL2.256; rows 32-byte aligned, launch_k checks):
// the k/4 lanes of a row cover a whole 128-byte X line per instruction -- half the L1
// wavefronts of 128-bit loads (the gather-bound pipe kernel runs L1TEX at 98 %)
template <int VEC>
__device__ __forceinline__ void ld_x(const double* __restrict__ p, double (&x)[VEC]) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
        for (int t = 0; t < VEC; t += 4)
            asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(x[t]), "=d"(x[t + 1]), "=d"(x[t + 2]), "=d"(x[t + 3])
                         : "l"(p + t));
    } else {
#pragma unroll
        for (int t = 0; t < VEC; t += 2) {
            double2 v = __ldg(reinterpret_cast<const double2*>(p) + t / 2);
            x[t] = v.x;
            x[t + 1] = v.y;
        }
    }
}

template <int VEC>
__device__ __forceinline__ void st_y(double* p, const double (&v)[VEC], int valid) {
    if (VEC >= 2 && valid == VEC) {
#pragma unroll
        for (int t = 0; t < VEC; t += 2) __stcs(reinterpret_cast<double2*>(p) + t / 2, make_double2(v[t], v[t + 1]));
    } else {
#pragma unroll
        for (int t = 0; t < VEC; ++t)
            if (t < valid) __stcs(p + t, v[t]);
    }
}

template <bool GHOST>
__device__ __forceinline__ const double* xrow(const SpmmArgs& a, int c) {
    return (GHOST && c >= a.ncol_local) ? a.Xg + (int64_t)(c - a.ncol_local) * a.ldg : a.X + (int64_t)c * a.ldx;
}

// acc += sum_{p in [s,e)} val[p] * X[col[p], c0 : c0+VEC], in CSR order, gathers batched
template <int VEC, bool GHOST>
__device__ __forceinline__ void row_accumulate(const SpmmArgs& a, const int* col, const double* val, int s, int e,
                                               int c0, bool lane_in, double (&acc)[VEC]) {
    constexpr int kBatch = Batch<VEC>::B;
    for (int p = s; p < e; p += kBatch) {
        double x[kBatch][VEC];
        double v[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            if (p + u < e && lane_in) {
                const int c = col[p + u];
                v[u] = val[p + u];
                ld_x(xrow<GHOST>(a, c) + c0, x[u]);
            } else {
                v[u] = 0.0;
#pragma unroll
                for (int t = 0; t < VEC; ++t) x[u][t] = 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
#pragma unroll
            for (int t = 0; t < VEC; ++t) acc[t] = fma(v[u], x[u][t], acc[t]);
    }
}

// out = acc C (C from shared memory via a per-row scratch line) or acc; then
// Y = alpha out + beta Y.  Every lane of the warp must call it (__syncwarp).
template <int KP, int VEC, bool HAS_C>
__device__ __forceinline__ void row_epilogue(const SpmmArgs& a, const double* s_C, double* t_row, int c0,
                                             bool active, int64_t row, const double (&acc)[VEC]) {
    const int k = a.k, kout = a.kout;
    double out[VEC];
    if (HAS_C) {
#pragma unroll
        for (int t = 0; t < VEC; ++t) t_row[c0 + t] = (c0 + t < k) ? acc[t] : 0.0;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < VEC; ++t) out[t] = 0.0;
        for (int c = 0; c < k; ++c) {
            const double tv = t_row[c];
#pragma unroll
            for (int t = 0; t < VEC; ++t) out[t] = fma(tv, s_C[c * KP + c0 + t], out[t]);
        }
        __syncwarp();
    } else {
#pragma unroll
        for (int t = 0; t < VEC; ++t) out[t] = acc[t];
    }
    if (active && c0 < kout) {
        double* yp = a.Y + row * a.ldy + c0;
        const int valid = min(VEC, kout - c0);
        double v[VEC];
        if (a.beta != 0.0) {
#pragma unroll
            for (int t = 0; t < VEC; ++t) v[t] = (t < valid) ? a.alpha * out[t] + a.beta * yp[t] : 0.0;
        } else {
#pragma unroll
            for (int t = 0; t < VEC; ++t) v[t] = a.alpha * out[t];
        }
        st_y<VEC>(yp, v, valid);
    }
}

template <int KP, bool HAS_C>
__device__ __forceinline__ void load_C(const SpmmArgs& a, double* s_C, int tid, int nthreads) {
    if (HAS_C) {
        for (int i = tid; i < KP * KP; i += nthreads) {
            const int r = i / KP, c = i % KP;
            s_C[i] = (r < a.k && c < a.kout) ? a.C[r * a.kout + c] : 0.0;
        }
    }
}

// All passes over one tile's rows (NC consumer threads).  Called separately
// with shared-memory and with global col/val pointers so the compiler emits
// LDS (not generic loads) for the staged case.
template <int KP, int VEC, bool HAS_C, int NC = kThreads, int TR = kTileRows>
__device__ __forceinline__ void tile_rows(const SpmmArgs& a, const int* col, const double* val, const int* s_rp,
                                          int nr, int64_t r0, int grp, int c0, bool lane_in, const double* s_C,
                                          double* t_row) {
    constexpr int RPP = NC / (KP / VEC);
    constexpr int PASSES = (TR + RPP - 1) / RPP;
#pragma unroll 1
    for (int pass = 0; pass < PASSES; ++pass) {
        const int r = pass * RPP + grp;
        const bool active = r < nr;
        double acc[VEC];
#pragma unroll
        for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
        if (active) row_accumulate<VEC, false>(a, col, val, s_rp[r], s_rp[r + 1], c0, lane_in, acc);
        row_epilogue<KP, VEC, HAS_C>(a, s_C, t_row, c0, active, r0 + r, acc);
    }
}

// ------------------------------------------------------------------ persistent TMA pipeline
// NC consumer threads, NS ring stages, MINB CTAs per SM (variants: DESIGN.md §4.1)
// Coupled apply on the FP64 tensor cores for the gather (pipe) kernel: each warp's rows of a
// pass (32 / LANES of them) go to a per-warp scratch (TS doubles per row), then
// Y(rows) = alpha (A X)(rows) C + beta Y as m8n8k4 DMMA with C as B fragments
// ([ks][nb][lane] in shared memory); blocks of 8 rows, rows beyond the warp's share are zero.
template <int KP>
struct CfRegs { static constexpr int N = (KP <= 16 && KP >= 8) ? (KP / 4) * (KP / 8) : 1; };

template <int KP, int VEC, int NC, int TR>
__device__ __forceinline__ void tile_rows_tce(const SpmmArgs& a, const int* col, const double* val, const int* s_rp,
                                              int nr, int64_t r0, int grp, int c0, bool lane_in,
                                              const double* s_Cf, const double (&cf)[CfRegs<KP>::N], double* w_scr) {
    constexpr int NCF = CfRegs<KP>::N;
    constexpr int LANES = KP / VEC;
    constexpr int RPP = NC / LANES;
    constexpr int PASSES = (TR + RPP - 1) / RPP;
    constexpr int WR = 32 / LANES;                  // rows per warp per pass
    constexpr int PP = WR < 8 ? 8 / WR : 1;         // passes per DMMA block (k > 16: 2, full m8 blocks)
    constexpr int NR = PP * WR, NB8 = (NR + 7) / 8; // scratch rows, 8-row DMMA blocks
    constexpr int NQ = KP / 4, NKO = KP / 8, TS = KP + 2;
    const int lane32 = threadIdx.x & 31, mg = lane32 >> 2, kq = lane32 & 3;
    const int lrow = lane32 / LANES;                // row of this lane inside the warp's share
    const int wrow0 = grp - lrow;                   // first group index of the warp
#pragma unroll 1
    for (int pass0 = 0; pass0 < PASSES; pass0 += PP) {
#pragma unroll
        for (int q = 0; q < PP; ++q) {
            const int r = (pass0 + q) * RPP + grp;
            const bool active = pass0 + q < PASSES && r < nr;
            double acc[VEC];
#pragma unroll
            for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
            if (active) row_accumulate<VEC, false>(a, col, val, s_rp[r], s_rp[r + 1], c0, lane_in, acc);
            double* tp = w_scr + (q * WR + lrow) * TS + c0;
            const bool keep = active && lane_in;
            reinterpret_cast<double2*>(tp)[0] = keep ? make_double2(acc[0], acc[1]) : make_double2(0.0, 0.0);
            reinterpret_cast<double2*>(tp)[1] = keep ? make_double2(acc[2], acc[3]) : make_double2(0.0, 0.0);
        }
        __syncwarp();
#pragma unroll
        for (int b = 0; b < NB8; ++b) {
            const int lr = 8 * b + mg;                  // scratch row of the fragment
            const bool rv = lr < NR;
            double af[NQ];
#pragma unroll
            for (int ks = 0; ks < NQ; ++ks) af[ks] = rv ? w_scr[lr * TS + 4 * ks + kq] : 0.0;
            const int pq = pass0 + lr / WR;
            const int row = pq * RPP + wrow0 + lr % WR;
            double dd[NKO][2];   // k-step outer: NKO independent accumulator chains
#pragma unroll
            for (int nb = 0; nb < NKO; ++nb) dd[nb][0] = dd[nb][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < NQ; ++ks)
#pragma unroll
                for (int nb = 0; nb < NKO; ++nb)
                    dmma(dd[nb][0], dd[nb][1], af[ks],
                         KP <= 16 ? cf[(ks * NKO + nb) % NCF] : s_Cf[(ks * NKO + nb) * 32 + lane32]);
#pragma unroll
            for (int nb = 0; nb < NKO; ++nb) {
                const double d0 = dd[nb][0], d1 = dd[nb][1];
                const int c = 8 * nb + 2 * kq;
                if (rv && pq < PASSES && row < nr && c < a.kout) {
                    double* yp = a.Y + (r0 + row) * a.ldy + c;
                    double v0 = a.alpha * d0, v1 = a.alpha * d1;
                    if (a.beta != 0.0) {
                        v0 = fma(a.beta, yp[0], v0);
                        if (c + 1 < a.kout) v1 = fma(a.beta, yp[1], v1);
                    }
                    if (c + 1 < a.kout) __stcs(reinterpret_cast<double2*>(yp), make_double2(v0, v1));
                    else __stcs(yp, v0);
                }
            }
        }
        __syncwarp();                                   // scratch reused by the next passes
    }
}

template <int NC, int NS, int MINB, int TR_, int CAP_>
struct PipeCfg {
    static constexpr int TR = TR_, CAP = CAP_;
    static constexpr int RP_INTS = TR + 8;                 // rows + 1, aligned start/end slack
    static constexpr int COL_INTS = CAP + 8;
    static constexpr int VAL_DBL = CAP + 8;
    static constexpr int RP_BYTES = RP_INTS * 4;
    static constexpr int COL_BYTES = COL_INTS * 4;
    static constexpr int VAL_BYTES = VAL_DBL * 8;
    static constexpr int STAGE_BYTES = RP_BYTES + COL_BYTES + VAL_BYTES;
    // ring + barriers/meta + (C and one scratch line per row group when coupled)
    static constexpr int bytes(int kp, int rpp, bool has_c) {
        // (TCE: C fragments = kp*kp doubles, per-warp scratch of max(32/lanes, 8) rows of kp+2:
        // <= max(rpp, 8 warps) rows)
        return NS * STAGE_BYTES + 64 * 8 + (has_c ? (kp * kp + (rpp > 8 * (NC / 32) ? rpp : 8 * (NC / 32)) * (kp + 2)) * 8 : 0);
    }
};

// processing-order tile t -> tile index (y-slab order, SpmmArgs::sl_*); identity if sl_S == 0
__device__ __forceinline__ int slab_tile(const SpmmArgs& a, int t) {
    if (a.sl_S <= 0) return t;
    const int per_plane = a.sl_L * a.sl_tpl, per_slab = a.sl_nz * per_plane;
    const int s = t / per_slab, rem = t - s * per_slab;
    const int z = rem / per_plane, rem2 = rem - z * per_plane;
    const int yl = rem2 / a.sl_tpl, xb = rem2 - yl * a.sl_tpl;
    return ((z * a.sl_ny + s * a.sl_L + yl) * a.sl_tpl) + xb;
}

template <int KP, int VEC, bool HAS_C, int NC, int NS, int MINB, int TR, int CAP>
__global__ void __launch_bounds__(NC + 32, MINB)
bspmm_pipe_kernel(const SpmmArgs a, int ntiles) {
    using L = PipeCfg<NC, NS, MINB, TR, CAP>;
    // tiles interleaved over the persistent CTAs (optionally permuted: slab_tile)
    const int tb = (int)blockIdx.x, te = ntiles, tstep = (int)gridDim.x;
    constexpr int LANES = KP / VEC;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * L::STAGE_BYTES);
    uint64_t* empty = full + NS;
    int* s_staged = reinterpret_cast<int*>(empty + NS);
    double* s_C = reinterpret_cast<double*>(smem + NS * L::STAGE_BYTES + 64 * 8);
    double* s_t = s_C + KP * KP;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    constexpr bool TCE = HAS_C && KP >= 8 && VEC == 4;
    if constexpr (TCE) {   // C as m8n8k4 B fragments [ks][nb][lane]
        constexpr int NQ = KP / 4, NKO = KP / 8;
        for (int i = tid; i < NQ * NKO * 32; i += NC + 32) {
            const int l = i & 31, ks = (i >> 5) / NKO, nb = (i >> 5) % NKO;
            const int r = 4 * ks + (l & 3), c = 8 * nb + (l >> 2);
            s_C[i] = (r < a.k && c < a.kout) ? a.C[r * a.kout + c] : 0.0;
        }
    } else {
        if (tid < NC) load_C<KP, HAS_C>(a, s_C, tid, NC);
    }
    __syncthreads();

    if (warp == NC / 32) {
        // ------------------------------------------------ producer warp
        if ((tid & 31) == 0) {
            const uint64_t pol = evict_first_policy();
            int i = 0;
            for (int tile = tb; tile < te; tile += tstep, ++i) {
                const int s = i % NS;
                if (i >= NS) mbar_wait(&empty[s], ((i / NS) - 1) & 1);
                unsigned char* st = smem + s * L::STAGE_BYTES;
                const int64_t r0 = a.row0 + (int64_t)slab_tile(a, tile) * TR;
                const int nr = (int)((a.row0 + a.nrows - r0) < TR ? (a.row0 + a.nrows - r0) : TR);
                const int p0 = a.rp[r0], p1 = a.rp[r0 + nr];
                const int64_t ra = r0 & ~(int64_t)3;
                const uint32_t rp_bytes = (uint32_t)((((r0 - ra) + nr + 1 + 3) & ~3) * 4);
                const bool staged = (p1 - p0) <= CAP;
                const int pa = p0 & ~3;
                const uint32_t n4 = (uint32_t)(((p0 - pa) + (p1 - p0) + 3) >> 2);
                s_staged[s] = staged ? 1 : 0;
                const uint32_t tx = rp_bytes + (staged && n4 ? n4 * 16u + n4 * 32u : 0u);
                mbar_expect_tx(&full[s], tx);
                bulk_g2s(st, a.rp + ra, rp_bytes, &full[s], pol);
                if (staged && n4) {
                    bulk_g2s(st + L::RP_BYTES, a.col + pa, n4 * 16u, &full[s], pol);
                    bulk_g2s(st + L::RP_BYTES + L::COL_BYTES, a.val + pa, n4 * 32u, &full[s], pol);
                }
            }
        }
        return;
    }
    // ---------------------------------------------------- consumer warps
    const int grp = tid / LANES, lane = tid % LANES, c0 = lane * VEC;
    const bool lane_in = c0 < a.k;
    double* t_row = s_t + grp * (KP + 1);
    // coupled k <= 16: C's B fragments in registers for the whole kernel
    double cf[CfRegs<KP>::N];
#pragma unroll
    for (int q = 0; q < CfRegs<KP>::N; ++q) cf[q] = (TCE && KP <= 16) ? s_C[q * 32 + (tid & 31)] : 0.0;
    int i = 0;
    for (int tile = tb; tile < te; tile += tstep, ++i) {
        const int s = i % NS;
        mbar_wait(&full[s], (i / NS) & 1);
        const unsigned char* st = smem + s * L::STAGE_BYTES;
        const int64_t r0 = a.row0 + (int64_t)slab_tile(a, tile) * TR;
        const int nr = (int)((a.row0 + a.nrows - r0) < TR ? (a.row0 + a.nrows - r0) : TR);
        const int roff = (int)(r0 & 3);
        const int* s_rp = reinterpret_cast<const int*>(st) + roff;
        const int p0 = s_rp[0];
        const int off = p0 & 3;
        const bool staged = s_staged[s] != 0;
        if constexpr (TCE) {
            double* w_scr = s_t + warp * ((32 / LANES) < 8 ? 8 : (32 / LANES)) * (KP + 2);
            if (staged) {
                const int* scol = reinterpret_cast<const int*>(st + L::RP_BYTES) + off - p0;
                const double* sval = reinterpret_cast<const double*>(st + L::RP_BYTES + L::COL_BYTES) + off - p0;
                tile_rows_tce<KP, VEC, NC, TR>(a, scol, sval, s_rp, nr, r0, grp, c0, lane_in, s_C, cf, w_scr);
            } else {
                tile_rows_tce<KP, VEC, NC, TR>(a, a.col, a.val, s_rp, nr, r0, grp, c0, lane_in, s_C, cf, w_scr);
            }
        } else if (staged) {
            const int* scol = reinterpret_cast<const int*>(st + L::RP_BYTES) + off - p0;
            const double* sval = reinterpret_cast<const double*>(st + L::RP_BYTES + L::COL_BYTES) + off - p0;
            tile_rows<KP, VEC, HAS_C, NC, TR>(a, scol, sval, s_rp, nr, r0, grp, c0, lane_in, s_C, t_row);
        } else {
            tile_rows<KP, VEC, HAS_C, NC, TR>(a, a.col, a.val, s_rp, nr, r0, grp, c0, lane_in, s_C, t_row);
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
}

template <int KP, int VEC, bool HAS_C, int NC, int NS, int MINB, int TR, int CAP>
void launch_pipe(const SpmmArgs& a, int num_sms, cudaStream_t st) {
    using L = PipeCfg<NC, NS, MINB, TR, CAP>;
    const int64_t ntiles = (a.nrows + TR - 1) / TR;
    const int smem = L::bytes(KP, NC / (KP / VEC), HAS_C);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(bspmm_pipe_kernel<KP, VEC, HAS_C, NC, NS, MINB, TR, CAP>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    const int64_t cap = (int64_t)MINB * (a.grid_sms > 0 && a.grid_sms < num_sms ? a.grid_sms : num_sms);
    const int64_t grid = ntiles < cap ? ntiles : cap;
    SpmmArgs b = a;
    if (b.sl_S > 0) {   // slab order needs whole tiles per line and a permutation of all tiles
        const int64_t line = (int64_t)b.sl_tpl;   // (host passed the line length here)
        if (line % TR != 0 || (int64_t)b.sl_ny * b.sl_nz * line != b.nrows || b.sl_ny % b.sl_S != 0) {
            b.sl_S = 0;
        } else {
            b.sl_tpl = (int)(line / TR);
            b.sl_L = b.sl_ny / b.sl_S;
        }
    }
    BK_KERNEL(bspmm_pipe_kernel<KP, VEC, HAS_C, NC, NS, MINB, TR, CAP><<<(unsigned)grid, NC + 32, smem, st>>>(
        b, (int)ntiles));
}

// ------------------------------------------------------------------ explicit row list
// Boundary rows of a partitioned matrix (ghost columns): no staging.
template <int KP, int VEC, bool HAS_C, bool GHOST>
__global__ void __launch_bounds__(kThreads)
bspmm_rows_kernel(const SpmmArgs a) {
    constexpr int LANES = KP / VEC;
    constexpr int RPP = kThreads / LANES;
    __shared__ double s_C[HAS_C ? KP * KP : 1];
    __shared__ double s_t[HAS_C ? RPP * (KP + 1) : 1];
    const int tid = threadIdx.x, grp = tid / LANES, lane = tid % LANES, c0 = lane * VEC;
    load_C<KP, HAS_C>(a, s_C, tid, kThreads);
    if (HAS_C) __syncthreads();
    const int64_t idx = (int64_t)blockIdx.x * RPP + grp;
    const bool active = idx < a.nrows;
    const int64_t row = active ? (a.rows ? (int64_t)a.rows[idx] : a.row0 + idx) : 0;
    double acc[VEC];
#pragma unroll
    for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
    if (active) row_accumulate<VEC, GHOST>(a, a.col, a.val, a.rp[row], a.rp[row + 1], c0, c0 < a.k, acc);
    row_epilogue<KP, VEC, HAS_C>(a, s_C, s_t + grp * (KP + 1), c0, active, row, acc);
}

// ------------------------------------------------------------------ dispatch
int num_sms_cached() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int KP, int VEC, bool HAS_C, bool GHOST>
void launch_t(const SpmmArgs& a, cudaStream_t st) {
    if (a.nrows <= 0) return;
    if (a.rows || GHOST) {
        constexpr int RPP = kThreads / (KP / VEC);
        const unsigned grid = (unsigned)((a.nrows + RPP - 1) / RPP);
        BK_KERNEL(bspmm_rows_kernel<KP, VEC, HAS_C, GHOST><<<grid, kThreads, 0, st>>>(a));
        return;
    }
    if constexpr (!GHOST) {
        // (round-1 A/B of ring depth / CTAs per SM / tile size: DESIGN.md §4.1)
        // (2 CTAs x 2 stages x 512-row tiles or 2 x 3 x 256 measured 15-45 % slower on c3 / c4:
        // the gathers need the third CTA's warps for latency hiding)
        // coupled k > 16: C's fragments and the per-warp DMMA scratch (25.6 KB) next to two
        // 256-row stages leave room for only TWO CTAs per SM (ncu c4 k = 32 coupled: warps active
        // 24 % vs 42 % plain, long-scoreboard 53 %: 4.96 ms vs 2.27 ms plain) -- 128-row tiles
        // keep the third CTA
        if constexpr (HAS_C && KP == 32)
            launch_pipe<KP, VEC, HAS_C, 256, 2, 3, 128, 1152>(a, num_sms_cached(), st);
        else
            launch_pipe<KP, VEC, HAS_C, 256, 2, 3, 256, 2304>(a, num_sms_cached(), st);
    }
}

template <int KP, int VEC>
void launch_kv(const SpmmArgs& a, cudaStream_t st) {
    const bool hc = a.C != nullptr, gh = a.Xg != nullptr;
    if (hc) {
        if (gh) launch_t<KP, VEC, true, true>(a, st); else launch_t<KP, VEC, true, false>(a, st);
    } else {
        if (gh) launch_t<KP, VEC, false, true>(a, st); else launch_t<KP, VEC, false, false>(a, st);
    }
}

// columns per thread: VEC = 4 when 256-bit gathers are legal (32-byte aligned X rows, k and
// k_out multiples of 4), else 2 (16-byte) or 1
template <int KP>
void launch_k(const SpmmArgs& a, cudaStream_t st, bool vec2) {
    const bool al32 = ((uintptr_t)a.X % 32 == 0) && (a.ldx % 4 == 0) &&
                      (a.Xg == nullptr || (((uintptr_t)a.Xg % 32 == 0) && a.ldg % 4 == 0));
    if constexpr (KP == 16) {
        // k = 12: three 4-column lanes per row (KP = 16 would leave one lane of four idle in
        // the gather-bound loop); 288 consumers = 96 rows per pass, 288-row tiles = 3 passes
        if (vec2 && al32 && a.k == 12 && a.kout == 12 && !a.C && !a.Xg && !a.rows && a.nrows > 0) {
            launch_pipe<12, 4, false, 288, 2, 3, 288, 2592>(a, num_sms_cached(), st);
            return;
        }
    }
    if constexpr (KP == 32) {
        // k = 24: six 4-column lanes per row (KP = 32 leaves two lanes of eight idle); same
        // 288-consumer / 288-row shape as k = 12 (48 rows per pass, 6 passes)
        if (vec2 && al32 && a.k == 24 && a.kout == 24 && !a.C && !a.Xg && !a.rows && a.nrows > 0) {
            launch_pipe<24, 4, false, 288, 2, 3, 288, 2592>(a, num_sms_cached(), st);
            return;
        }
        // k = 20: five lanes per row; 320 consumers = 64 rows per pass, two CTAs per SM with a
        // three-stage ring (three 352-thread CTAs would cap the kernel at 62 registers)
        if (vec2 && al32 && a.k == 20 && a.kout == 20 && !a.C && !a.Xg && !a.rows && a.nrows > 0) {
            launch_pipe<20, 4, false, 320, 3, 2, 256, 2304>(a, num_sms_cached(), st);
            return;
        }
    }
    if constexpr (KP >= 4) {
        if (vec2 && al32 && a.k % 4 == 0 && a.kout % 4 == 0) return launch_kv<KP, 4>(a, st);
    }
    if constexpr (KP >= 2) {
        if (vec2) return launch_kv<KP, 2>(a, st);
    }
    launch_kv<KP, 1>(a, st);
}


// ------------------------------------------------------------------ windowed pipeline (X staged in shared memory)
// DESIGN.md §4.1.  For a band-structured matrix (every nonzero on a few
// diagonals d = col - row, bk_plan_bands) the X rows a tile of rows [r0, r0+T)
// needs are one contiguous segment per band, [r0 + lo_g, r0 + T + hi_g).  The
// producer warp moves the tile's CSR ranges AND those segments into a shared-
// memory ring with TMA bulk copies (no per-tile plan: addresses follow from r0;
// only the tile's two row-pointer bounds are prefetched, several tiles ahead,
// with cp.async); the consumers' gathers become shared-memory loads.  Column-
// chunk order alternates between rows so the 16-byte LDS of a warp spread over
// all 32 banks.
struct BandArgs {
    SpmmArgs a;
    int lo[BK_BAND_MAX], hi[BK_BAND_MAX], wb[BK_BAND_MAX];   // segment bounds, window row base
    int G;              // bands
    int TR, cap, ns;    // rows per tile, staged nonzeros per tile, ring stages
    int stage_bytes, off_col, off_val, off_rp;
    int ntiles;
    int64_t ncols;      // rows of X
    // fused reduction epilogue (RED > 0; the fused block-BiCGStab passes): the
    // rows [r0, r0 + nr) of e[0] (= Rt) and e[1] (= R) are staged with the tile, and
    //   RED 1:  ro.blk[0][0] = e0^T Y, ro.blk[0][1] = e0^T e1         (Y = A X, e.g. V = A P)
    //   RED 2:  ro.blk[0][0] = e0^T Y, dots[0] = <Y_c, X_c>, dots[1] = <Y_c, Y_c>   (T = A S)
    //   RED 3:  ro.blk[0][0] = X^T Y (X from the staged window; no extra operand)   (Q = A P)
    //   RED 4:  ro.blk[0][0] = X^T Y, ro.blk[0][1] = X^T X (X from the window)      (W = A R, O11)
    // are accumulated on the FP64 tensor cores / in FMA registers and reduced over the grid in
    // a fixed order (reduce.cuh); the CTA that writes the result runs the k x k epilogue `epi`.
    const double* e[2];
    int off_e[2];
    RedOut ro;
    SmallEpi epi;
    int pf;             // L2 prefetch distance in tiles of this CTA (0: off)
};
constexpr int kMetaDepth = 8;   // tiles whose row-pointer bounds are in flight

// One X row chunk (VEC doubles at column c0) of window row `wr`.
template <int VEC>
__device__ __forceinline__ void win_load(const double* xp, int sw, double (&x)[VEC]) {
    if constexpr (VEC == 4) {
        const double2 lo = reinterpret_cast<const double2*>(xp)[sw];
        const double2 hi = reinterpret_cast<const double2*>(xp)[1 - sw];
        x[0] = lo.x; x[1] = lo.y; x[2] = hi.x; x[3] = hi.y;
    } else if constexpr (VEC == 2) {
        const double2 q = *reinterpret_cast<const double2*>(xp);
        x[0] = q.x; x[1] = q.y;
    } else {
#pragma unroll
        for (int t = 0; t < VEC; ++t) x[t] = xp[t];
    }
}

// acc += sum_{p in [s,e)} val[p] X[col[p], cols] with X from the staged window (window row of
// column c: c + fo[g] for the last band g with c >= thr[g]).  MR > 0: every row has <= MR
// nonzeros (the plan's bound), one branch-free pass with clamped indices and zero weights;
// MR == 0: batches of 4.  Column sets: VEC consecutive columns at c0 (16-byte chunks in the
// order sw), or (SPLIT, k > 16) the chunks at cA and cB = cA + 16: the 8 lanes of a row then
// read 128 contiguous bytes per LDS.128 -- one wavefront per row, no bank conflicts (the
// consecutive-column map read 16-byte chunks 32 bytes apart: 2-way conflicts).
// Lanes whose columns lie beyond k compute on in-bounds garbage that is never stored.
template <int VEC, int NB, int MR, bool SPLIT = false>
__device__ __forceinline__ void band_accumulate(const double* s_win, const int* col, const double* val, int s, int e,
                                                const int (&thr)[NB], const int (&fo)[NB], int kk, int c0, int sw,
                                                double (&acc)[VEC]) {
    constexpr int B = MR > 0 ? MR : 4;
    for (int p = s; p < e; p += B) {
        double x[B][VEC];
        double v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int q = (p + u < e) ? p + u : e - 1;
            const int c = col[q];
            v[u] = (p + u < e) ? val[q] : 0.0;
            int f = fo[0];
#pragma unroll
            for (int g = 1; g < NB; ++g) f = (c >= thr[g]) ? fo[g] : f;
            if constexpr (SPLIT) {
                const double* xr = s_win + (c + f) * kk + c0;
                const double2 lo = *reinterpret_cast<const double2*>(xr);
                const double2 hi = *reinterpret_cast<const double2*>(xr + 16);
                x[u][0] = lo.x; x[u][1] = lo.y; x[u][2] = hi.x; x[u][3] = hi.y;
            } else {
                win_load<VEC>(s_win + (c + f) * kk + c0, sw, x[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u)
#pragma unroll
            for (int t = 0; t < VEC; ++t) acc[t] = fma(v[u], x[u][t], acc[t]);
        if constexpr (MR > 0) break;
    }
    if constexpr (VEC == 4 && !SPLIT) {
        if (sw) {   // chunks were accumulated in swapped order
            const double t0 = acc[0], t1 = acc[1];
            acc[0] = acc[2]; acc[1] = acc[3]; acc[2] = t0; acc[3] = t1;
        }
    }
}

// Y[row, cA:cA+2] and Y[row, cB:cB+2] = alpha acc + beta Y (SPLIT column map, no coupling)
__device__ __forceinline__ void store_split(const SpmmArgs& a, int64_t row, int cA, int cB, const double (&acc)[4]) {
    const int cs[2] = {cA, cB};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = cs[h];
        if (c >= a.kout) continue;
        double* yp = a.Y + row * a.ldy + c;
        double v0 = a.alpha * acc[2 * h], v1 = a.alpha * acc[2 * h + 1];
        if (a.beta != 0.0) {
            v0 = fma(a.beta, yp[0], v0);
            v1 = fma(a.beta, yp[1], v1);
        }
        __stcs(reinterpret_cast<double2*>(yp), make_double2(v0, v1));
    }
}

template <int KP, int VEC, bool HAS_C, int NC, int NB, int MR, bool KEXACT, int RED = 0>
__global__ void __launch_bounds__(NC + 32, RED ? 2 : 1)   // (fused reduction: keep 2 CTAs per SM)
bspmm_win_kernel(const BandArgs w) {
    static_assert(RED == 0 || (!HAS_C && VEC == 4 && (KP == 8 || KP == 16)), "fused reduction: plain apply, k 8..16");
    constexpr int NE = RED == 1 ? 2 : (RED == 2 ? 1 : 0);   // streamed extra operands
    const SpmmArgs& a = w.a;
    constexpr int LANES = KP / VEC;
    constexpr int RPP = NC / LANES;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + w.ns * w.stage_bytes);
    uint64_t* empty = full + 8;
    int2* s_pp = reinterpret_cast<int2*>(empty + 8);           // kMetaDepth row-pointer bounds
    double* s_C = reinterpret_cast<double*>(s_pp + kMetaDepth);
    double* s_t = s_C + KP * KP;
    // coupled apply on the FP64 tensor cores (TCE): C as m8n8k4 B fragments [ks][nb][lane],
    // then the tile's (A X) rows (TS doubles per row) for the DMMA epilogue
    constexpr bool TCE = HAS_C && KP >= 8 && VEC == 4;
    constexpr int NQ = KP / 4, NKO = KP / 8, TS = KP + 2;
    double* s_Cf = s_C;
    double* s_tT = s_Cf + NQ * NKO * 32;

    const int tid = threadIdx.x, warp = tid >> 5, lane32 = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < w.ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC / 32);
        }
        mbar_fence_init();
    }
    if constexpr (TCE) {
        for (int i = tid; i < NQ * NKO * 32; i += blockDim.x) {
            const int l = i & 31, ks = (i >> 5) / NKO, nb = (i >> 5) % NKO;
            const int r = 4 * ks + (l & 3), c = 8 * nb + (l >> 2);
            s_Cf[i] = (r < a.k && c < a.kout) ? a.C[r * a.kout + c] : 0.0;
        }
    } else {
        if (tid < NC) load_C<KP, HAS_C>(a, s_C, tid, NC);
    }
    __syncthreads();

    const int k = a.k;
    if (warp == NC / 32) {
        // ------------------------------------------------ producer (one thread)
        if (lane32 != 0) return;
        const uint64_t pol_once = evict_first_policy();    // CSR: read once
        const uint64_t pol_x = evict_normal_policy();      // X rows: re-read by the neighbouring tiles
        const int64_t rend = a.row0 + a.nrows;
        auto fetch = [&](int tile, int slot) {
            if (tile < w.ntiles) {
                const int64_t r0 = a.row0 + (int64_t)tile * w.TR;
                const int64_t r1 = (rend - r0) < w.TR ? rend : r0 + w.TR;
                const uint32_t dst = smem_u32(s_pp + slot);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(a.rp + r0) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4), "l"(a.rp + r1) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        for (int d = 0; d < kMetaDepth; ++d) fetch(blockIdx.x + d * gridDim.x, d);
        const uint32_t kb = (uint32_t)k * 8u;
        int s = 0, slot = 0;
        uint32_t ph = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < w.ntiles; tile += gridDim.x, ++i) {
            int2 pq = make_int2(0, 0);   // row-pointer bounds of the tile prefetched (w.pf == 1)
            if (w.pf == 1) {
                asm volatile("cp.async.wait_group %0;" ::"n"(kMetaDepth - 2) : "memory");
                pq = s_pp[slot + 1 == kMetaDepth ? 0 : slot + 1];
            } else {
                asm volatile("cp.async.wait_group %0;" ::"n"(kMetaDepth - 1) : "memory");
            }
            const int2 pp = s_pp[slot];
            fetch(tile + kMetaDepth * gridDim.x, slot);
            slot = (slot + 1 == kMetaDepth) ? 0 : slot + 1;
            if (i >= w.ns) mbar_wait(&empty[s], ph ^ 1u);
            unsigned char* st = smem + s * w.stage_bytes;
            double* s_win = reinterpret_cast<double*>(st);
            const int64_t r0 = a.row0 + (int64_t)tile * w.TR;
            const int nr = (int)((rend - r0) < w.TR ? (rend - r0) : w.TR);
            const int p0 = pp.x, p1 = pp.y;
            const int64_t ra = r0 & ~(int64_t)3;
            const uint32_t rp_bytes = (uint32_t)((((r0 - ra) + nr + 1 + 3) & ~3) * 4);
            const int pc = p0 & ~3, pv = p0 & ~1;
            const uint32_t col_bytes = p1 > p0 ? (uint32_t)(((p1 - pc + 3) & ~3) * 4) : 0u;
            const uint32_t val_bytes = p1 > p0 ? (uint32_t)(((p1 - pv + 1) & ~1) * 8) : 0u;
            uint32_t bytes = rp_bytes + col_bytes + val_bytes;
            int64_t sa[NB];
            uint32_t sb[NB];
#pragma unroll
            for (int g = 0; g < NB; ++g) {
                sb[g] = 0;
                sa[g] = 0;
                if (g < w.G) {
                    const int64_t lo = r0 + w.lo[g];
                    const int64_t a0 = lo < 0 ? 0 : lo;
                    int64_t b0 = r0 + nr + w.hi[g];
                    if (b0 > w.ncols) b0 = w.ncols;
                    if (b0 > a0) {
                        uint32_t b = (uint32_t)(b0 - a0) * kb;
                        double* dst = s_win + (int64_t)(w.wb[g] + (a0 - lo)) * k;
                        if (b & 15u) {   // odd k and X ends at an odd row: last row by hand
                            b -= kb;
                            const double* src = a.X + (b0 - 1) * k;
                            double* d1 = dst + (b0 - 1 - a0) * k;
                            for (int t = 0; t < k; ++t) d1[t] = src[t];
                            // generic stores into a stage that later ring phases fill
                            // through the async proxy (cp.async.bulk): order them
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        }
                        sa[g] = a0;
                        sb[g] = b;
                        bytes += b;
                    }
                }
            }
            if constexpr (NE > 0) bytes += (uint32_t)NE * (uint32_t)nr * kb;
            mbar_expect_tx(&full[s], bytes);
            bulk_g2s(st + w.off_rp, a.rp + ra, rp_bytes, &full[s], pol_once);
            if (col_bytes) {
                bulk_g2s(st + w.off_col, a.col + pc, col_bytes, &full[s], pol_once);
                bulk_g2s(st + w.off_val, a.val + pv, val_bytes, &full[s], pol_once);
            }
#pragma unroll
            for (int g = 0; g < NB; ++g) {
                if (sb[g]) {
                    const int64_t lo = r0 + w.lo[g];
                    bulk_g2s(s_win + (int64_t)(w.wb[g] + (sa[g] - lo)) * k, a.X + sa[g] * k, sb[g], &full[s], pol_x);
                }
            }
            if constexpr (NE > 0) {   // the tile's rows of Rt (and R): read once
#pragma unroll
                for (int j = 0; j < NE; ++j)
                    bulk_g2s(st + w.off_e[j], w.e[j] + r0 * k, (uint32_t)nr * kb, &full[s], pol_once);
            }
            // L2 prefetch of what this CTA's tile pf tiles ahead reads from DRAM first: its
            // leading band segment (the other bands were fetched by earlier tiles), its rows of
            // the streamed operands and (pf == 1) its CSR ranges -- the ring's stages then wait
            // on L2, not on DRAM
            const int t2 = tile + w.pf * (int)gridDim.x;
            if (w.pf > 0 && t2 < w.ntiles) {
                const int64_t q0 = a.row0 + (int64_t)t2 * w.TR;
                const int nq = (int)((rend - q0) < w.TR ? (rend - q0) : w.TR);
                if constexpr (NE > 0) {
#pragma unroll
                    for (int j = 0; j < NE; ++j) bulk_prefetch_l2(w.e[j] + q0 * k, (uint32_t)nq * kb);
                }
                const int g = w.G - 1;
                const int64_t lo = q0 + w.lo[g];
                const int64_t a0 = lo < 0 ? 0 : lo;
                int64_t b0 = q0 + nq + w.hi[g];
                if (b0 > w.ncols) b0 = w.ncols;
                const uint32_t xb = b0 > a0 ? ((uint32_t)(b0 - a0) * kb) & ~15u : 0u;
                if (xb) bulk_prefetch_l2(a.X + a0 * k, xb);
                if (w.pf == 1 && pq.y > pq.x) {
                    const int qc = pq.x & ~3, qv = pq.x & ~1;
                    bulk_prefetch_l2(a.col + qc, (uint32_t)(((pq.y - qc + 3) & ~3) * 4));
                    bulk_prefetch_l2(a.val + qv, (uint32_t)(((pq.y - qv + 1) & ~1) * 8));
                }
            }
            if (++s == w.ns) {
                s = 0;
                ph ^= 1u;
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        return;
    }
    // ---------------------------------------------------- consumer warps
    // column map: VEC consecutive columns at c0, or (SPLIT: k > 16, 8 lanes per row) the
    // 16-byte chunks at cA = 2 lane and cB = cA + 16 (conflict-free window loads)
    constexpr bool SPLIT = KP == 32 && VEC == 4;
    const int grp = tid / LANES, lane = tid % LANES, c0 = SPLIT ? 2 * lane : lane * VEC;
    const int cA = c0, cB = SPLIT ? c0 + 16 : c0 + 2;
    const int kk = KEXACT ? KP : k;
    double* t_row = s_t + grp * (KP + 1);
    const int passes = (w.TR + RPP - 1) / RPP;
    // coupled (TCE): WR rows per warp and pass; k > 16 has WR = 4, so PP = 2 passes fill one
    // 8-row DMMA block (half-empty blocks doubled the epilogue's tensor-core work)
    constexpr int WR = 32 / LANES;
    constexpr int PP = (TCE && WR < 8) ? 8 / WR : 1;
    // (C's fragments stay in shared memory here: register-resident fragments raised the k = 16
    // kernel to 106 registers and measured 0.66 -> 0.49 of HBM; the gather kernel keeps them)
    // fused reduction (RED): Gram fragments (m8n8k4 accumulators) and per-lane column dots
    constexpr int RNA = KP / 8;
    constexpr bool TWO = RED == 1 || RED == 4;   // two k x k blocks
    double g0[RED ? RNA : 1][RED ? RNA : 1][2], g1[TWO ? RNA : 1][TWO ? RNA : 1][2];
    double dd0[RED == 2 ? 4 : 1], dd1[RED == 2 ? 4 : 1];
    if constexpr (RED > 0) {
#pragma unroll
        for (int i = 0; i < RNA; ++i)
#pragma unroll
            for (int j = 0; j < RNA; ++j) {
                g0[i][j][0] = g0[i][j][1] = 0.0;
                if constexpr (TWO) g1[i][j][0] = g1[i][j][1] = 0.0;
            }
        if constexpr (RED == 2)
#pragma unroll
            for (int t = 0; t < 4; ++t) dd0[t] = dd1[t] = 0.0;
    }
    // Y(rows) = alpha (A X)(rows) C + beta Y as m8n8k4 DMMA by the warp itself over its NR scratch
    // rows (no CTA barrier, so the other warps keep gathering); rowof(lr, grow)
    // gives scratch row lr's global row and whether it is stored
    auto tce_epi = [&](auto&& rowof) {
        if constexpr (TCE) {
            constexpr int NR = PP * WR, NB8 = (NR + 7) / 8;
            const double* w_scr = s_tT + warp * NR * TS;
            __syncwarp();
            const int mg = lane32 >> 2, kq = lane32 & 3;
#pragma unroll
            for (int b = 0; b < NB8; ++b) {
                const int lr = 8 * b + mg;
                int64_t grow = 0;
                const bool rv = lr < NR && rowof(lr, grow);
                double af[NQ];
#pragma unroll
                for (int ks = 0; ks < NQ; ++ks) af[ks] = rv ? w_scr[lr * TS + 4 * ks + kq] : 0.0;
                // k-step outer, output block inner: NKO independent accumulator chains in
                // flight instead of one dependent chain of NQ DMMAs per output block
                double dd[NKO][2];
#pragma unroll
                for (int nb = 0; nb < NKO; ++nb) dd[nb][0] = dd[nb][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < NQ; ++ks)
#pragma unroll
                    for (int nb = 0; nb < NKO; ++nb)
                        dmma(dd[nb][0], dd[nb][1], af[ks], s_Cf[(ks * NKO + nb) * 32 + lane32]);
#pragma unroll
                for (int nb = 0; nb < NKO; ++nb) {
                    const double d0 = dd[nb][0], d1 = dd[nb][1];
                    const int c = 8 * nb + 2 * kq;
                    if (rv && c < a.kout) {
                        double* yp = a.Y + grow * a.ldy + c;
                        double v0 = a.alpha * d0, v1 = a.alpha * d1;
                        if (a.beta != 0.0) {
                            v0 = fma(a.beta, yp[0], v0);
                            if (c + 1 < a.kout) v1 = fma(a.beta, yp[1], v1);
                        }
                        if (c + 1 < a.kout) __stcs(reinterpret_cast<double2*>(yp), make_double2(v0, v1));
                        else __stcs(yp, v0);
                    }
                }
            }
            __syncwarp();
        }
    };
    // coupled k > 16 with one pass per tile (TR <= RPP, e.g. k = 32 on 64-row tiles): a DMMA
    // block pairs the warp's rows of TWO consecutive tiles of this CTA (scratch halves xq = 0, 1;
    // each stage is released right after its gathers) instead of padding every block with a
    // second, empty pass (half the epilogue's tensor-core work was on zero rows)
    const bool xt = TCE && PP == 2 && passes == 1;
    int xq = 0;
    int64_t xr0a = 0, xr0b = 0;   // (scalars: a dynamically indexed pair would live in local memory)
    int xnra = 0, xnrb = 0;
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < w.ntiles; tile += gridDim.x) {
        mbar_wait(&full[s], ph);
        const unsigned char* st = smem + s * w.stage_bytes;
        const int64_t r0 = a.row0 + (int64_t)tile * w.TR;
        const int nr = (int)((a.row0 + a.nrows - r0) < w.TR ? (a.row0 + a.nrows - r0) : w.TR);
        const int* s_rp = reinterpret_cast<const int*>(st + w.off_rp) + (int)(r0 & 3);
        const int p0 = s_rp[0];
        const int* scol = reinterpret_cast<const int*>(st + w.off_col) + (p0 & 3) - p0;
        const double* sval = reinterpret_cast<const double*>(st + w.off_val) + (p0 & 1) - p0;
        const double* s_win = reinterpret_cast<const double*>(st);
        // window row of column c: c + fo[g] for the last band g with c >= thr[g]
        int thr[NB], fo[NB];
#pragma unroll
        for (int g = 0; g < NB; ++g) {
            const bool on = g < w.G;
            thr[g] = on ? (int)(r0 + w.lo[g]) : INT_MAX;
            fo[g] = on ? (int)(w.wb[g] - (r0 + w.lo[g])) : 0;
        }
        if constexpr (TCE && PP == 2) {
            if (xt) {
                const int r = grp;   // the tile's single pass
                const bool active = r < nr;
                double acc[VEC];
#pragma unroll
                for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
                if (active) {
                    const int rs = s_rp[r], re = s_rp[r + 1];
                    if (re > rs) {
                        const int gr = (int)(r0 + r);
                        const int sw = (kk <= 16) ? (((gr * kk) >> 4) & 1) : (gr & 1);
                        band_accumulate<VEC, NB, MR, SPLIT>(s_win, scol, sval, rs, re, thr, fo, kk, c0, sw, acc);
                    }
                }
                double* tp = s_tT + warp * (PP * WR) * TS + (xq * WR + lane32 / LANES) * TS;
                reinterpret_cast<double2*>(tp + cA)[0] =
                    (active && cA < a.k) ? make_double2(acc[0], acc[1]) : make_double2(0.0, 0.0);
                reinterpret_cast<double2*>(tp + cB)[0] =
                    (active && cB < a.k) ? make_double2(acc[2], acc[3]) : make_double2(0.0, 0.0);
                if (xq) { xr0b = r0; xnrb = nr; } else { xr0a = r0; xnra = nr; }
                __syncwarp();
                if (lane32 == 0) mbar_arrive(&empty[s]);   // the scratch holds what the epilogue needs
                if (xq == 1) {
                    tce_epi([&](int lr, int64_t& grow) {
                        const int h = lr / WR, row = warp * WR + lr % WR;
                        grow = (h ? xr0b : xr0a) + row;
                        return row < (h ? xnrb : xnra);
                    });
                }
                xq ^= 1;
                if (++s == w.ns) {
                    s = 0;
                    ph ^= 1u;
                }
                continue;
            }
        }
#pragma unroll 1
        for (int pass0 = 0; pass0 < passes; pass0 += PP) {
#pragma unroll
            for (int q = 0; q < PP; ++q) {
                const int pass = pass0 + q;
                const int r = pass * RPP + grp;
                const bool active = pass < passes && r < nr;
                double acc[VEC];
#pragma unroll
                for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
                if (active) {
                    const int rs = s_rp[r], re = s_rp[r + 1];
                    if (re > rs) {
                        const int gr = (int)(r0 + r);
                        const int sw = (kk <= 16) ? (((gr * kk) >> 4) & 1) : (gr & 1);
                        band_accumulate<VEC, NB, MR, SPLIT>(s_win, scol, sval, rs, re, thr, fo, kk, c0, sw, acc);
                    }
                }
                if constexpr (TCE) {
                    // this warp's rows -> its scratch (columns >= k zero: C's padded rows are
                    // zero, and 0 x garbage could be NaN)
                    double* w_scr = s_tT + warp * (PP * WR) * TS;
                    const int lrow = q * WR + lane32 / LANES;
                    double* tp = w_scr + lrow * TS;
                    reinterpret_cast<double2*>(tp + cA)[0] =
                        (active && cA < a.k) ? make_double2(acc[0], acc[1]) : make_double2(0.0, 0.0);
                    reinterpret_cast<double2*>(tp + cB)[0] =
                        (active && cB < a.k) ? make_double2(acc[2], acc[3]) : make_double2(0.0, 0.0);
                } else if constexpr (SPLIT) {
                    if (active) store_split(a, r0 + r, cA, cB, acc);
                } else {
                    row_epilogue<KP, VEC, HAS_C>(a, s_C, t_row, c0, active, r0 + r, acc);
                }
                if constexpr (RED > 0) {
                    // the warp's WR rows of Y -> its scratch (columns >= k and inactive rows zero)
                    double* w_scr = s_C + warp * WR * TS;
                    double* tp = w_scr + (lane32 / LANES) * TS + c0;
                    const bool keep = active && c0 < k;
                    reinterpret_cast<double2*>(tp)[0] = keep ? make_double2(acc[0], acc[1]) : make_double2(0.0, 0.0);
                    reinterpret_cast<double2*>(tp)[1] = keep ? make_double2(acc[2], acc[3]) : make_double2(0.0, 0.0);
                    if constexpr (RED == 2) {   // <Y_c, X_c>, <Y_c, Y_c>: X row r from the staged window
                        if (keep) {
                            const int c = (int)(r0 + r);
                            int f = fo[0];
#pragma unroll
                            for (int g = 1; g < NB; ++g) f = (c >= thr[g]) ? fo[g] : f;
                            const double* xr = s_win + (int64_t)(c + f) * kk + c0;
                            const double2 xa = reinterpret_cast<const double2*>(xr)[0];
                            const double2 xb = reinterpret_cast<const double2*>(xr)[1];
                            const double xv[4] = {xa.x, xa.y, xb.x, xb.y};
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                dd0[t] = fma(acc[t], xv[t], dd0[t]);
                                dd1[t] = fma(acc[t], acc[t], dd1[t]);
                            }
                        }
                    }
                    __syncwarp();
                    // e0^T Y (and e0^T e1) over the warp's rows: blocks of 8 rows, two k-steps of 4
                    const int mg = lane32 >> 2, kq = lane32 & 3;
                    const double* E0 = reinterpret_cast<const double*>(st + w.off_e[0]);
                    const double* E1 = reinterpret_cast<const double*>(st + w.off_e[RED == 1 ? 1 : 0]);
                    // RED 3 (X^T Y, e.g. P^T Q of block CG): the left operand is the apply's own
                    // input, read from the staged window (centre row of each tile row)
#pragma unroll
                    for (int b = 0; b < WR / 8; ++b)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int lr = 8 * b + 4 * h + kq;               // scratch row (k index)
                            const int tr = pass * RPP + warp * WR + lr;      // tile row
                            const bool rin = pass < passes && tr < nr;
                            double af[RNA], bf[RNA], cf[RED == 1 ? RNA : 1];
                            const double* erow = E0 + (int64_t)tr * k;
                            if constexpr (RED >= 3) {
                                const int c = (int)(r0 + tr);
                                int f = fo[0];
#pragma unroll
                                for (int g = 1; g < NB; ++g) f = (c >= thr[g]) ? fo[g] : f;
                                erow = s_win + (int64_t)(c + f) * kk;
                            }
#pragma unroll
                            for (int i = 0; i < RNA; ++i) {
                                const int col = 8 * i + mg;
                                const bool ok = rin && col < k;
                                af[i] = ok ? erow[col] : 0.0;
                                bf[i] = ok ? w_scr[lr * TS + col] : 0.0;
                                if constexpr (RED == 1) cf[i] = ok ? E1[(int64_t)tr * k + col] : 0.0;
                            }
#pragma unroll
                            for (int i = 0; i < RNA; ++i)
#pragma unroll
                                for (int j = 0; j < RNA; ++j) {
                                    dmma(g0[i][j][0], g0[i][j][1], af[i], bf[j]);
                                    if constexpr (RED == 1) dmma(g1[i][j][0], g1[i][j][1], af[i], cf[j]);
                                    if constexpr (RED == 4) dmma(g1[i][j][0], g1[i][j][1], af[i], af[j]);
                                }
                        }
                    __syncwarp();
                }
            }
            if constexpr (TCE) {
                tce_epi([&](int lr, int64_t& grow) {
                    const int row = (pass0 + lr / WR) * RPP + warp * WR + lr % WR;
                    grow = r0 + row;
                    return pass0 + lr / WR < passes && row < nr;
                });
            }
        }
        __syncwarp();
        if (lane32 == 0) mbar_arrive(&empty[s]);   // the stage is no longer read

        if (++s == w.ns) {
            s = 0;
            ph ^= 1u;
        }
    }
    if constexpr (TCE && PP == 2) {
        if (xt && xq == 1) {   // an odd number of tiles: the last half pairs with nothing
            tce_epi([&](int lr, int64_t& grow) {
                const int row = warp * WR + lr % WR;
                grow = xr0a + row;
                return lr < WR && row < xnra;
            });
        }
    }
    if constexpr (RED > 0) {
        // every issued copy was waited on: once all consumers are here the ring holds the combine
        constexpr int KBP = (TWO ? 2 : 1) * KP, NOUT = KP * KBP + 64;
        asm volatile("bar.sync 1, %0;" ::"r"(NC));
        double* s_red = reinterpret_cast<double*>(smem);
        const int mg = lane32 >> 2, kq = lane32 & 3;
        // grid_reduce reads output (a, b) at a * KBP + b with the Y blocks packed k apart
        // (b = block * k + c): columns >= k of a block are padding and are not written
#pragma unroll
        for (int i = 0; i < RNA; ++i)
#pragma unroll
            for (int j = 0; j < RNA; ++j) {
                const int c = 8 * j + 2 * kq;
                if (c >= k) continue;
                double* d = s_red + warp * NOUT + (8 * i + mg) * KBP + c;
                d[0] = g0[i][j][0];
                d[1] = g0[i][j][1];
                if constexpr (TWO) {
                    d[k] = g1[i][j][0];
                    d[k + 1] = g1[i][j][1];
                }
            }
        if constexpr (RED == 2) {
            // lanes holding the same columns (equal lane % LANES): fixed xor tree
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int m = LANES; m < 32; m <<= 1) {
                    dd0[t] += __shfl_xor_sync(0xffffffffu, dd0[t], m);
                    dd1[t] += __shfl_xor_sync(0xffffffffu, dd1[t], m);
                }
            if (lane32 < LANES)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    s_red[warp * NOUT + NOUT - 64 + c0 + t] = dd0[t];
                    s_red[warp * NOUT + NOUT - 32 + c0 + t] = dd1[t];
                }
        }
        const int kb_real = (TWO ? 2 : 1) * k;
        if (grid_reduce<NC, NOUT>(w.ro, s_red, k * kb_real + (RED == 2 ? 2 * k : 0), kb_real, KBP, false) &&
            w.epi.kind && warp == 0)
            dd::run_small_epi(w.epi, reinterpret_cast<double*>(smem));
    }
}


// the fused reduction of one launch (RED > 0): extra operands, outputs, k x k epilogue
struct RedArgs {
    const double* e0;
    const double* e1;
    RedOut ro;
    const SmallEpi* epi;
};

template <int KP, int VEC, bool HAS_C, int NB, int MR, bool KEXACT, int NC, int RED = 0>
bool launch_win_t(const SpmmArgs& a, const BandPlan& p, cudaStream_t st, int ctas, bool big_tiles = true,
                  const RedArgs* ra = nullptr) {
    constexpr int LANES = KP / VEC;
    constexpr int RPP = NC / LANES;
    static const int tr_env = env_int("BK_WIN_TR", 0);
    BandArgs w{};
    w.a = a;
    w.G = p.nbands;
    // L2 prefetch one tile ahead (A/B, profiles/r02/e19_prefetch.txt, c2): RED 1 / 2 at k = 16
    // 139 / 127 -> 132 / 119 us, k = 8 75 / 71 -> 73 / 68 us; plain apply k = 8 / 16 37.9 / 64.5 ->
    // 35.8 / 62.5 us.  Off where it measured slower: RED 3 (111 -> 116 us), plain k = 32 (129 ->
    // 142 us: the 8-lane rows already keep enough bytes in flight), coupled applies.
    static const int pf_red = env_int("BK_RED_PF", -1), pf_win = env_int("BK_WIN_PF", -1);
    const int pf_dflt = ((RED == 1 || RED == 2) || (RED == 0 && !HAS_C && (KP == 8 || KP == 16))) ? 1 : 0;
    w.pf = RED > 0 ? (pf_red >= 0 ? pf_red : pf_dflt) : (HAS_C ? 0 : (pf_win >= 0 ? pf_win : pf_dflt));
    if constexpr (RED > 0) {
        w.e[0] = ra->e0;
        w.e[1] = ra->e1;
        w.ro = ra->ro;
        if (ra->epi) w.epi = *ra->epi;
    }
    auto r16 = [](int64_t x) { return (x + 15) & ~(int64_t)15; };
    auto layout = [&](int TR) {
        w.TR = TR;
        w.cap = TR * p.max_row_nnz;
        int wrows = 0;
        for (int g = 0; g < p.nbands; ++g) {
            w.lo[g] = p.lo[g];
            w.hi[g] = p.hi[g];
            w.wb[g] = wrows;
            wrows += TR + p.hi[g] - p.lo[g];
        }
        const int64_t win = (int64_t)wrows * a.k * 8;
        w.off_col = (int)r16(win);
        w.off_val = w.off_col + (int)r16((int64_t)(w.cap + 4) * 4);
        w.off_rp = w.off_val + (int)r16((int64_t)(w.cap + 2) * 8);
        int end = w.off_rp + (int)r16((TR + 8) * 4);
        for (int j = 0; j < (RED == 1 ? 2 : (RED == 2 ? 1 : 0)); ++j) {   // staged rows of Rt (, R)
            w.off_e[j] = end;
            end += (int)r16((int64_t)TR * a.k * 8);
        }
        w.stage_bytes = (int)((end + 127) & ~(int64_t)127);
    };
    // barriers + row-pointer ring + (C, coupled-apply scratch): with the tensor-core epilogue
    // (TCE) C fragments and the per-warp (A X) rows (RPP rows of KP + 2), else C and one
    // scratch line per row group
    constexpr bool TCE = HAS_C && KP >= 8 && VEC == 4;
    auto fixed_for = [&](int tr) {
        // TCE scratch: (NC / 32) warps x max(WR, 8) rows (k > 16 pairs two passes per warp)
        constexpr int scr_rows = (NC / 32) * ((32 / LANES) < 8 ? 8 : (32 / LANES));
        (void)tr;
        const int cb = TCE ? ((KP / 4) * (KP / 8) * 32 + scr_rows * (KP + 2)) * 8
                           : (RED ? RPP * (KP + 2) : KP * KP + (HAS_C ? RPP * (KP + 1) : 0)) * 8;
        return 16 * 8 + kMetaDepth * 8 + cb;
    };
    // two CTAs per SM: half the shared memory each (the fused-reduction kernels also hold a few
    // bytes of static shared memory: 1 KB less)
    constexpr int kHalf = (RED ? 112 : 113) * 1024;
    // (coupled k > 16 pairs PP passes per DMMA block: a tile holds at least PP passes)
    constexpr int PPm = (TCE && (32 / LANES) < 8) ? 8 / (32 / LANES) : 1;
    int TR = std::max(64, PPm * RPP);
    if (tr_env > 0) {
        TR = std::max(2, tr_env & ~1);
    } else if (ctas == 2 && big_tiles) {   // the largest multiple of 16 rows with two stages per CTA
        // (fused reductions: a multiple of the RPP rows of one pass, so no pass runs its DMMA
        // epilogue on mostly empty row blocks -- c2 k = 16 RED 2 with 80-row tiles (64 + 16-row
        // passes) 131 us, with 64-row tiles 124 us)
        const int step = (RED > 0 && RPP >= 16) ? RPP : 16;
        for (int t = (std::min(1024, 8 * RPP) / step) * step; t >= 64; t -= step) {
            layout(t);
            if (2 * w.stage_bytes + fixed_for(t) <= kHalf) {
                TR = t;
                break;
            }
        }
    }
    layout(TR);
    int fixed = fixed_for(TR);
    int budget = (ctas == 1 ? 227 * 1024 : kHalf) - fixed;
    while (budget / w.stage_bytes < 2 && TR > 2 * 2) {   // huge windows: smaller tiles
        TR = (TR / 2) & ~1;
        layout(TR);
        fixed = fixed_for(TR);
        budget = (ctas == 1 ? 227 * 1024 : kHalf) - fixed;
    }
    int ns = budget / w.stage_bytes;
    if (ns > 8) ns = 8;
    if (ns < 2) return false;
    w.ns = ns;
    if constexpr (RED > 0) {   // the combine buffer (warps x NOUT doubles) reuses the drained ring
        constexpr int KBP = (RED == 1 || RED == 4 ? 2 : 1) * KP;
        if ((size_t)(NC / 32) * (KP * KBP + 64) * 8 > (size_t)ns * w.stage_bytes) return false;
    }
    const int64_t ntiles = (a.nrows + w.TR - 1) / w.TR;
    if (ntiles >= (1ll << 31)) return false;
    w.ntiles = (int)ntiles;
    w.ncols = a.ncol_local;
    const int smem = ns * w.stage_bytes + fixed;
    // the exact dynamic size (the fused-reduction instantiations also hold static shared memory,
    // so "227 KB dynamic" would be refused); raised when a later launch needs more
    static int attr_bytes = 0;
    if (smem > attr_bytes) {
        cudaFuncSetAttribute(bspmm_win_kernel<KP, VEC, HAS_C, NC, NB, MR, KEXACT, RED>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_bytes = smem;
    }
    const int nsm = num_sms_cached();
    const int64_t cap = (int64_t)ctas * (a.grid_sms > 0 && a.grid_sms < nsm ? a.grid_sms : nsm);
    const int64_t grid = ntiles < cap ? ntiles : cap;
    BK_KERNEL(bspmm_win_kernel<KP, VEC, HAS_C, NC, NB, MR, KEXACT, RED><<<(unsigned)grid, NC + 32, smem, st>>>(w));
    return true;
}

// CTA shape: two 256-consumer CTAs per SM when each still gets >= 3 ring
// stages in half the shared memory, else one CTA with 512 consumers (more
// warps for latency hiding, full shared memory for the window).  Env
// BK_WIN_CTAS=1|2 forces it (A/B).
template <int KP, int VEC, bool HAS_C, int NB, int MR, bool KEXACT>
bool launch_win_shape(const SpmmArgs& a, const BandPlan& p, cudaStream_t st) {
    static const int force = env_int("BK_WIN_CTAS", 0);
    // two CTAs per SM with the largest tile that keeps 2 stages each (launch_win_t); measured
    // against one 512-thread CTA and RPP-row tiles: c2 k = 4 / 8 / 16 0.63 / 0.79 / 0.74 ->
    // 0.77 / 0.81 / 0.81 of HBM (tile 256 / 192 / 112 rows)
    int ctas = (force == 1 || force == 2) ? force : 2;
    if (force != 1 && force != 2 && HAS_C) {
        // coupled applies keep the earlier shape rule (3 stages of RPP-row tiles in 100 KB ->
        // 2 CTAs, else one 512-thread CTA): c2 k = 4 / 16 coupled 0.63 / 0.64 vs 0.48 / 0.60
        const int rpp = 256 / (KP / VEC), tr = rpp < 64 ? 64 : rpp;
        int64_t wrows = 0;
        for (int g = 0; g < p.nbands; ++g) wrows += tr + p.hi[g] - p.lo[g];
        const int64_t stage = wrows * a.k * 8 + (int64_t)tr * p.max_row_nnz * 12 + tr * 4 + 256;
        ctas = (3 * stage <= 100 * 1024) ? 2 : 1;
        if (ctas == 2) return launch_win_t<KP, VEC, HAS_C, NB, MR, KEXACT, 256>(a, p, st, 2, false);
    }
    if (ctas == 1 && KP >= 4) return launch_win_t<KP, VEC, HAS_C, NB, MR, KEXACT, 512>(a, p, st, 1);
    return launch_win_t<KP, VEC, HAS_C, NB, MR, KEXACT, 256>(a, p, st, ctas);
}

template <int KP, int VEC, bool HAS_C, int NB, int MR>
bool launch_win_ke(const SpmmArgs& a, const BandPlan& p, cudaStream_t st) {
    return a.k == KP ? launch_win_shape<KP, VEC, HAS_C, NB, MR, true>(a, p, st)
                     : launch_win_shape<KP, VEC, HAS_C, NB, MR, false>(a, p, st);
}

// 2-D 5-point (3 bands, <= 5 nonzeros per row), 3-D 7-point (5 bands, <= 7),
// anything else band structured: 7 bands, batched rows
template <int KP, int VEC, bool HAS_C>
bool launch_win_nb(const SpmmArgs& a, const BandPlan& p, cudaStream_t st) {
    if (p.nbands <= 3 && p.max_row_nnz <= 5) return launch_win_ke<KP, VEC, HAS_C, 3, 5>(a, p, st);
    if (p.nbands <= 5 && p.max_row_nnz <= 7) return launch_win_ke<KP, VEC, HAS_C, 5, 7>(a, p, st);
    return launch_win_ke<KP, VEC, HAS_C, BK_BAND_MAX, 0>(a, p, st);
}

template <int KP, int VEC>
bool launch_win_kv(const SpmmArgs& a, const BandPlan& p, cudaStream_t st) {
    return a.C ? launch_win_nb<KP, VEC, true>(a, p, st) : launch_win_nb<KP, VEC, false>(a, p, st);
}

template <int KP>
bool launch_win_k(const SpmmArgs& a, const BandPlan& p, cudaStream_t st, bool vec2) {
    if constexpr (KP >= 4) {
        if (vec2 && a.k % 4 == 0 && a.kout % 4 == 0) return launch_win_kv<KP, 4>(a, p, st);
    }
    if constexpr (KP >= 2) {
        if (vec2) return launch_win_kv<KP, 2>(a, p, st);
    }
    if constexpr (KP <= 8) return launch_win_kv<KP, 1>(a, p, st);   // odd k: one column per lane
    return false;
}

bool win_enabled() {
    static const int v = env_int("BK_SPMM_WIN", 1);
    return v != 0;
}

}  // namespace

void launch_bspmm(const SpmmArgs& a, cudaStream_t st) {
    const int kmax = a.k > a.kout ? a.k : a.kout;
    // 16-byte vector path: even widths, even leading dims, 16-byte aligned bases
    bool vec2 = (a.k % 2 == 0) && (a.kout % 2 == 0) && (a.ldx % 2 == 0) && (a.ldy % 2 == 0) &&
                ((uintptr_t)a.X % 16 == 0) && ((uintptr_t)a.Y % 16 == 0) &&
                (a.Xg == nullptr || (((uintptr_t)a.Xg % 16 == 0) && a.ldg % 2 == 0));
    if (kmax <= 1) launch_k<1>(a, st, false);
    else if (kmax <= 2) launch_k<2>(a, st, vec2);
    else if (kmax <= 4) launch_k<4>(a, st, vec2);
    else if (kmax <= 8) launch_k<8>(a, st, vec2);
    else if (kmax <= 16) launch_k<16>(a, st, vec2);
    else launch_k<32>(a, st, vec2);
}

bool launch_bspmm_win_red(const SpmmArgs& a, const BandPlan& p, cudaStream_t st, int red, const double* e0,
                          const double* e1, const RedOut& ro, const SmallEpi* epi) {
    if (!win_enabled() || red < 1 || red > 4) return false;
    // 2-D 5-point lattices (3 bands), plain apply, k = 8, 12, 16, packed and 16-byte aligned operands
    if (p.nbands != 3 || p.max_row_nnz > 5 || a.C || a.rows || a.Xg || a.alpha != 1.0 || a.beta != 0.0) return false;
    if (a.row0 != p.row0 || a.nrows != p.nrows || a.nrows <= 0) return false;
    const int k = a.k;
    if (!(k == 8 || k == 12 || k == 16) || a.kout != k || a.ldx != k || a.ldy != k) return false;
    auto al16 = [](const void* q) { return q && ((uintptr_t)q & 15) == 0; };
    if (!al16(a.X) || !al16(a.Y) || (red <= 2 && !al16(e0)) || (red == 1 && !al16(e1))) return false;
    RedArgs ra{e0, e1, ro, epi};
    ra.ro.mode = 2;
    ra.ro.ka = k;
    ra.ro.kb = (red == 1 || red == 4 ? 2 : 1) * k;
    ra.ro.kw = k;
#define BK_RED(KP_, KX)                                                                              \
    switch (red) {                                                                               \
        case 1: return launch_win_t<KP_, 4, false, 3, 5, KX, 256, 1>(a, p, st, 2, true, &ra);   \
        case 2: return launch_win_t<KP_, 4, false, 3, 5, KX, 256, 2>(a, p, st, 2, true, &ra);   \
        case 4: return launch_win_t<KP_, 4, false, 3, 5, KX, 256, 4>(a, p, st, 2, true, &ra);   \
        default: return launch_win_t<KP_, 4, false, 3, 5, KX, 256, 3>(a, p, st, 2, true, &ra);  \
    }
    if (k == 8) { BK_RED(8, true) }
    if (k == 16) { BK_RED(16, true) }
    BK_RED(16, false)
#undef BK_RED
}

bool launch_bspmm_win(const SpmmArgs& a, const BandPlan& p, cudaStream_t st) {
    if (!win_enabled() || p.nbands <= 0 || a.rows || a.Xg) return false;
    // 3-D lattices (5 bands): the plain apply is faster with L1 gathers (pipe kernel,
    // c4 k = 16: 0.66 vs 0.57 of HBM) -- staging 5 band segments fills shared memory
    // with L2-hit bytes; the coupled apply keeps the DMMA tile epilogue
    // The same holds for k > 16 on 2-D lattices once the gathers are 256-bit loads (c2 k = 32:
    // 0.65 vs 0.63, k = 24: 0.54 vs 0.49; the band kernel is shared-memory bound there,
    // L1TEX 83 %).
    static const int wc = env_int("BK_WIN_COUPLED", 1);
    if (a.C != nullptr && !wc) return false;
    // k = 12 (e.g. 3 stages x 4 steps): the band kernel pads it to four 4-column lanes with a
    // run-time row stride; the gather kernel has a three-lane instantiation (launch_k) -- c2 plain
    // 83.0 vs 58.4 us (0.49 vs 0.70 of HBM), coupled 119 vs 87 us (profiles/r02/head/e22_*).
    // (k = 24 / 20, plain: the six- / five-lane gather instantiations, A/B knobs BK_WIN_K24 / K20)
    static const int w24 = env_int("BK_WIN_K24", 0), w20 = env_int("BK_WIN_K20", 0);
    if (((!w24 && a.k == 24 && a.kout == 24) || (!w20 && a.k == 20 && a.kout == 20)) && !a.C && a.ldx % 4 == 0 && ((uintptr_t)a.X % 32) == 0 &&
        a.ldy % 2 == 0 && ((uintptr_t)a.Y % 16) == 0)
        return false;
    static const int w12 = env_int("BK_WIN_K12", 0);
    if (!w12 && a.k == 12 && a.kout == 12 && a.ldx % 4 == 0 && ((uintptr_t)a.X % 32) == 0 && a.ldy % 2 == 0 &&
        ((uintptr_t)a.Y % 16) == 0)
        return false;
    static const int w3 = env_int("BK_WIN_3D", -1);
    // Coupled applies (per-warp DMMA epilogue in both kernels) follow the same rule: c2 k = 16
    // 0.64 band vs 0.52 gather, c4 k = 8 / 16 0.71 / 0.53 gather vs 0.63 / 0.49 band.
    // k > 16 on 2-D lattices: the conflict-free split column map (SPLIT) -- A/B: BK_WIN_3D=0
    if (w3 < 0 && p.nbands >= 5) return false;
    if (w3 == 0 && a.k > 16) return false;
    if (a.row0 != p.row0 || a.nrows != p.nrows || a.nrows <= 0) return false;
    // the window copies contiguous X rows: packed X (ldx == k), 16-byte aligned
    if (a.ldx != a.k || ((uintptr_t)a.X % 16) != 0) return false;
    const int kmax = a.k > a.kout ? a.k : a.kout;
    const bool vec2 = (a.k % 2 == 0) && (a.kout % 2 == 0) && (a.ldy % 2 == 0) && ((uintptr_t)a.Y % 16 == 0);
    if (kmax <= 1) return launch_win_k<1>(a, p, st, false);
    if (kmax <= 2) return launch_win_k<2>(a, p, st, vec2);
    if (kmax <= 4) return launch_win_k<4>(a, p, st, vec2);
    if (kmax <= 8) return launch_win_k<8>(a, p, st, vec2);
    if (kmax <= 16) return launch_win_k<16>(a, p, st, vec2);
    return launch_win_k<32>(a, p, st, vec2);
}

}  // namespace bk
