// stream.cu -- TMA-staged streaming kernels for the N x k passes of the block
// Krylov iteration (a3 Gram, a5 update, column dots) on sm_100a.
//
// The block vectors are row-major with ld == width, so a tile of T rows of
// each operand is ONE contiguous range: a producer warp moves it HBM -> shared
// memory with a single cp.async.bulk per operand (mbarrier complete_tx, 2-stage
// ring, persistent grid of 2 CTAs per SM), which keeps ~100 KB per SM in
// flight -- the memory-level parallelism the plain per-thread loads lacked
// (profiles/).  Eight consumer warps compute from shared memory:
//   update : out = a Xin + s P C + w W          (C in shared memory, FMA)
//   gram   : G  = X^T Y  on the FP64 tensor cores (mma.sync m8n8k4, DMMA),
//            per-CTA partial + last-CTA fixed-order reduction (deterministic)
//   coldot : d_c = sum_r X[r,c] Y[r,c] (+ d2 with Y2), same reduction scheme.
// Tiles whose byte count is not a multiple of 16 (only a ragged last tile can
// be) are read directly from global memory by the consumers.
#include "bk_internal.h"
#include "ptx.cuh"
#include "dense_dev.cuh"
#include "reduce.cuh"

#ifndef BK_STREAM_NSTAGE
#define BK_STREAM_NSTAGE 2
#endif
#ifndef BK_STREAM_STAGE_KB
#define BK_STREAM_STAGE_KB 48
#endif

namespace bk {
namespace {

constexpr int NC = 256;            // consumer threads
constexpr int NSTAGE = BK_STREAM_NSTAGE;
constexpr int STAGE_BYTES = BK_STREAM_STAGE_KB * 1024;


// Up to 3 contiguous row-major operands streamed tile by tile.
constexpr int MAXS = 5;            // operands per stream tile
struct Streams {
    const double* p[MAXS];
    int w[MAXS];     // doubles per row (0 = unused)
    int off[MAXS];   // byte offset of the operand inside a stage
    int nin;
    int T;           // rows per tile
    int64_t n;
    int ntiles;
};

__device__ __forceinline__ void stream_setup(uint64_t* full, uint64_t* empty) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
}

// producer warp, lane 0: returns after the last tile is issued
__device__ __forceinline__ void stream_produce(const Streams& S, unsigned char* smem, uint64_t* full, uint64_t* empty,
                                               int* s_direct) {
    const uint64_t pol = evict_first_policy();
    int i = 0;
    for (int tile = blockIdx.x; tile < S.ntiles; tile += gridDim.x, ++i) {
        const int s = i % NSTAGE;
        if (i >= NSTAGE) mbar_wait(&empty[s], ((i / NSTAGE) - 1) & 1);
        const int64_t r0 = (int64_t)tile * S.T;
        const int nr = (int)((S.n - r0) < S.T ? (S.n - r0) : S.T);
        bool ok = true;
        uint32_t tx = 0;
        for (int j = 0; j < S.nin; ++j) {
            const uint32_t b = (uint32_t)nr * S.w[j] * 8u;
            if ((b & 15u) || (((uintptr_t)(S.p[j] + r0 * S.w[j])) & 15u)) ok = false;
            tx += b;
        }
        s_direct[s] = ok ? 0 : 1;
        mbar_expect_tx(&full[s], ok ? tx : 0u);
        if (ok) {
            unsigned char* st = smem + s * STAGE_BYTES;
            for (int j = 0; j < S.nin; ++j)
                if (S.w[j] > 0)
                    bulk_g2s(st + S.off[j], S.p[j] + r0 * S.w[j], (uint32_t)nr * S.w[j] * 8u, &full[s], pol);
        }
    }
}

// ------------------------------------------------------------------ update
// out[r, c] = a Xin[r, c] + s sum_q P[r, q] C[q, c] + wv W[r, c];  P, Xin, W contiguous.
struct UpdStream {
    Streams S;          // 0 = P (kp), 1 = Xin (k, if a != 0), 2 = W (k, if present)
    int iX, iW;         // stream index of Xin / W, -1 if absent
    int iP;             // stream index of P (-1 when kp == 0: out = a Xin + w W)
    int kp, k, cw;      // cw = columns per thread (1, 2 or 4)
    double a, s, w_host;
    const double* w_dev;
    const double* C;    // kp x k
    double* out;
    int64_t ldo;        // output leading dimension (>= k; inputs are contiguous)
    const int* halt;
};

// row-0 pointer of the P operand for one tile: staged (stage base st) or global (direct)
__device__ __forceinline__ const double* p_rows(const UpdStream& U, const unsigned char* st, int64_t r0, bool direct) {
    if (U.iP < 0) return nullptr;
    return direct ? U.S.p[U.iP] + r0 * U.kp : reinterpret_cast<const double*>(st + U.S.off[U.iP]);
}

template <int CW>
__device__ __forceinline__ void upd_tile(const UpdStream& U, const double* Pt, const double* Xt,
                                         const double* Wt, const double* sC, int nr, int64_t r0, double wv) {
    const int k = U.k, kp = U.kp;
    const int tpr = k / CW;
    for (int idx = threadIdx.x; idx < nr * tpr; idx += NC) {
        const int r = idx / tpr, cb = (idx - r * tpr) * CW;
        double acc[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) acc[j] = 0.0;
        if (Pt) {
            const double* pr = Pt + (int64_t)r * kp;
            for (int q = 0; q < kp; ++q) {
                const double p = pr[q];
#pragma unroll
                for (int j = 0; j < CW; ++j) acc[j] = fma(p, sC[q * k + cb + j], acc[j]);
            }
        }
        double o[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            double v = U.s * acc[j];
            if (Xt) v = fma(U.a, Xt[(int64_t)r * k + cb + j], v);
            if (Wt) v = fma(wv, Wt[(int64_t)r * k + cb + j], v);
            o[j] = v;
        }
        double* op = U.out + (r0 + r) * U.ldo + cb;
        if (CW == 4) {
            reinterpret_cast<double2*>(op)[0] = make_double2(o[0], o[1]);
            reinterpret_cast<double2*>(op)[1] = make_double2(o[2], o[3]);
        } else if (CW == 2) {
            reinterpret_cast<double2*>(op)[0] = make_double2(o[0], o[1]);
        } else {
            op[0] = o[0];
        }
    }
}

// Tensor-core tile: out(8-row block) = a X + w W + P (s C), P (8 x kp) as A
// fragments (m8n8k4: lane holds P[row 4g+.., q]), s C as B fragments held in
// registers for the whole kernel.  Needs k % 8 == 0 and kp % 4 == 0.
template <int NQ, int NK>
__device__ __forceinline__ void upd_tile_mma(const UpdStream& U, const double* Pt, const double* Xt,
                                             const double* Wt, const double (&bf)[NQ][NK], int nr, int64_t r0,
                                             double wv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, mg = lane >> 2;
    const int k = U.k, kp = U.kp;
    for (int rb = 8 * warp; rb < nr; rb += 8 * (NC / 32)) {
        const int r = rb + mg;
        const bool rin = r < nr;
        double af[NQ];
#pragma unroll
        for (int ks = 0; ks < NQ; ++ks) af[ks] = rin ? Pt[(int64_t)r * kp + 4 * ks + kq] : 0.0;
        __syncwarp();   // in place (out == P) on a direct tile: the row is read before any lane writes it
        // k <= 16: k-step outer, so the NK output blocks are independent DMMA chains in flight;
        // k > 16 (sC already holds 2 NQ NK registers): one output block at a time
        if constexpr (NQ * NK <= 8) {
            double dd[NK][2];
#pragma unroll
            for (int nb = 0; nb < NK; ++nb) {
                const int c = 8 * nb + 2 * kq;
                const bool cin = rin && c < k;   // (k % 8 == 4: the last block is half outside)
                double d0 = 0.0, d1 = 0.0;
                if (cin && Xt) {
                    const double2 x = *reinterpret_cast<const double2*>(Xt + (int64_t)r * k + c);
                    d0 = U.a * x.x;
                    d1 = U.a * x.y;
                }
                if (cin && Wt) {
                    const double2 w = *reinterpret_cast<const double2*>(Wt + (int64_t)r * k + c);
                    d0 = fma(wv, w.x, d0);
                    d1 = fma(wv, w.y, d1);
                }
                dd[nb][0] = d0;
                dd[nb][1] = d1;
            }
            // D(row = mg, cols 2kq, 2kq+1): the accumulator layout of m8n8k4
#pragma unroll
            for (int ks = 0; ks < NQ; ++ks)
#pragma unroll
                for (int nb = 0; nb < NK; ++nb) dmma(dd[nb][0], dd[nb][1], af[ks], bf[ks][nb]);
#pragma unroll
            for (int nb = 0; nb < NK; ++nb) {
                const int c = 8 * nb + 2 * kq;
                if (rin && c < k)
                    *reinterpret_cast<double2*>(U.out + (r0 + r) * U.ldo + c) = make_double2(dd[nb][0], dd[nb][1]);
            }
        } else {
#pragma unroll
            for (int nb = 0; nb < NK; ++nb) {
                const int c = 8 * nb + 2 * kq;
                const bool cin = rin && c < k;
                double d0 = 0.0, d1 = 0.0;
                if (cin && Xt) {
                    const double2 x = *reinterpret_cast<const double2*>(Xt + (int64_t)r * k + c);
                    d0 = U.a * x.x;
                    d1 = U.a * x.y;
                }
                if (cin && Wt) {
                    const double2 w = *reinterpret_cast<const double2*>(Wt + (int64_t)r * k + c);
                    d0 = fma(wv, w.x, d0);
                    d1 = fma(wv, w.y, d1);
                }
#pragma unroll
                for (int ks = 0; ks < NQ; ++ks) dmma(d0, d1, af[ks], bf[ks][nb]);
                if (cin) *reinterpret_cast<double2*>(U.out + (r0 + r) * U.ldo + c) = make_double2(d0, d1);
            }
        }
    }
}

template <int NQ, int NK>
__global__ void __launch_bounds__(NC + 32, 2) upd_stream_mma_kernel(const UpdStream U) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    if (U.halt && *U.halt) return;
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(U.S, smem, full, empty, s_direct);
        return;
    }
    // B fragments of s C: lane holds (sC)[4 ks + kq][8 nb + mg]
    double bf[NQ][NK];
#pragma unroll
    for (int ks = 0; ks < NQ; ++ks)
#pragma unroll
        for (int nb = 0; nb < NK; ++nb) {   // (k a multiple of 4: columns >= k are zero)
            const int oc = 8 * nb + (lane >> 2);
            bf[ks][nb] = oc < U.k ? U.s * U.C[(4 * ks + (lane & 3)) * U.k + oc] : 0.0;
        }
    const double wv = U.iW >= 0 ? (U.w_dev ? U.w_host * *U.w_dev : U.w_host) : 0.0;
    int i = 0;
    for (int tile = blockIdx.x; tile < U.S.ntiles; tile += gridDim.x, ++i) {
        const int s = i % NSTAGE;
        mbar_wait(&full[s], (i / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * U.S.T;
        const int nr = (int)((U.S.n - r0) < U.S.T ? (U.S.n - r0) : U.S.T);
        if (!s_direct[s]) {
            const unsigned char* st = smem + s * STAGE_BYTES;
            const double* Xt = U.iX >= 0 ? reinterpret_cast<const double*>(st + U.S.off[U.iX]) : nullptr;
            const double* Wt = U.iW >= 0 ? reinterpret_cast<const double*>(st + U.S.off[U.iW]) : nullptr;
            upd_tile_mma<NQ, NK>(U, p_rows(U, st, r0, false), Xt, Wt, bf, nr, r0, wv);
        } else {
            const double* Xt = U.iX >= 0 ? U.S.p[U.iX] + r0 * U.k : nullptr;
            const double* Wt = U.iW >= 0 ? U.S.p[U.iW] + r0 * U.k : nullptr;
            upd_tile_mma<NQ, NK>(U, p_rows(U, nullptr, r0, true), Xt, Wt, bf, nr, r0, wv);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

template <int CW>
__global__ void __launch_bounds__(NC + 32, 2) upd_stream_kernel(const UpdStream U) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    double* sC = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES + 128);
    if (U.halt && *U.halt) return;
    stream_setup(full, empty);
    for (int i = threadIdx.x; i < U.kp * U.k; i += blockDim.x) sC[i] = U.C[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp == NC / 32) {
        if ((threadIdx.x & 31) == 0) stream_produce(U.S, smem, full, empty, s_direct);
        return;
    }
    const double wv = U.iW >= 0 ? (U.w_dev ? U.w_host * *U.w_dev : U.w_host) : 0.0;
    int i = 0;
    for (int tile = blockIdx.x; tile < U.S.ntiles; tile += gridDim.x, ++i) {
        const int s = i % NSTAGE;
        mbar_wait(&full[s], (i / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * U.S.T;
        const int nr = (int)((U.S.n - r0) < U.S.T ? (U.S.n - r0) : U.S.T);
        if (!s_direct[s]) {
            const unsigned char* st = smem + s * STAGE_BYTES;
            const double* Xt = U.iX >= 0 ? reinterpret_cast<const double*>(st + U.S.off[U.iX]) : nullptr;
            const double* Wt = U.iW >= 0 ? reinterpret_cast<const double*>(st + U.S.off[U.iW]) : nullptr;
            upd_tile<CW>(U, p_rows(U, st, r0, false), Xt, Wt, sC, nr, r0, wv);
        } else {
            const double* Xt = U.iX >= 0 ? U.S.p[U.iX] + r0 * U.k : nullptr;
            const double* Wt = U.iW >= 0 ? U.S.p[U.iW] + r0 * U.k : nullptr;
            upd_tile<CW>(U, p_rows(U, nullptr, r0, true), Xt, Wt, sC, nr, r0, wv);
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    }
}

// ------------------------------------------------------------------ gram (DMMA) / coldot
struct GramStream {
    Streams S;          // 0 = X (ka), 1 = Y (kb) (absent when X == Y), 2 = Y2 for coldot
    int ka, kb;
    int same;           // Y == X
    int y2x;            // coldot: Y2 == X (read from X's tile, not streamed twice)
    double* part;       // [gridDim.x][NOUT]
    int* ticket;
    double* G;          // gram: ka x kb; coldot: d[k]
    double* G2;         // coldot second output
    // multi-operand Gram (mode 2): X = [S.p[xs[0]] ... ], Y = [S.p[ys[0]] ...], every
    // array kw wide; output block (i, j) (kw x kw) goes to blk[i][j] (null = dropped)
    int mode;           // 0 gram, 1 coldot, 2 multi-operand gram
    int kw, nxa, nya;
    int xs[3], ys[2];
    double* blk[3][2];
    // mode 2 extra: column dots dots[q][c] = sum_r S.p[da[q]][r,c] * S.p[db[q]][r,c] (FMA, q < ndot)
    int ndot;
    int da[2], db[2];
    double* dots[2];
    // panel Gram (16-column panels): X panel p = columns [xpo[p], xpo[p] + 16) of stream xps[p]
    int nxp, nyp;
    int xps[4], xpo[4], yps[4], ypo[4];
    SmallEpi epi;       // k x k epilogue run by the CTA that writes the final result
};

// NSET independent accumulator sets (quads alternate between them) so the
// DMMA accumulation is not one long dependent chain per warp.
// (register cap 96 at 2 CTAs x 288 threads: more sets spill in the hot loop)
template <int NA, int NB>
struct GramSets { static constexpr int NSET = (NA * NB <= 2) ? 4 : ((NA * NB <= 4) ? 2 : 1); };

template <int NA, int NB>
__device__ __forceinline__ void gram_tile(const GramStream& Gs, const double* Xt, const double* Yt, int nr,
                                          double (&acc)[GramSets<NA, NB>::NSET][NA][NB][2]) {
    constexpr int NSET = GramSets<NA, NB>::NSET;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, mg = lane >> 2;
    const int ka = Gs.ka, kb = Gs.kb;
    for (int q0 = 4 * warp; q0 < nr; q0 += 4 * (NC / 32) * NSET) {
        double av[NSET][NA], bv[NSET][NB];
#pragma unroll
        for (int s = 0; s < NSET; ++s) {
            const int r = q0 + 4 * (NC / 32) * s + kq;
            const bool rin = r < nr;
#pragma unroll
            for (int i = 0; i < NA; ++i) av[s][i] = (rin && 8 * i + mg < ka) ? Xt[(int64_t)r * ka + 8 * i + mg] : 0.0;
#pragma unroll
            for (int j = 0; j < NB; ++j) bv[s][j] = (rin && 8 * j + mg < kb) ? Yt[(int64_t)r * kb + 8 * j + mg] : 0.0;
        }
#pragma unroll
        for (int s = 0; s < NSET; ++s)
#pragma unroll
            for (int i = 0; i < NA; ++i)
#pragma unroll
                for (int j = 0; j < NB; ++j) dmma(acc[s][i][j][0], acc[s][i][j][1], av[s][i], bv[s][j]);
    }
}

template <int NOUT>
__device__ __forceinline__ bool finish_reduce(const GramStream& Gs, double* s_red, int nout_real, int kb_real,
                                              int ld_out, bool coldot) {
    return grid_reduce<NC, NOUT>(Gs, s_red, nout_real, kb_real, ld_out, coldot);
}

// k x k epilogue (warp 0 of the final CTA), scratch = the drained ring
__device__ __forceinline__ void small_epilogue(const SmallEpi& e, unsigned char* smem) {
    if (e.kind && (threadIdx.x >> 5) == 0) dd::run_small_epi(e, reinterpret_cast<double*>(smem));
}

template <int NA, int NB>
__global__ void __launch_bounds__(NC + 32, 2) gram_stream_kernel(const GramStream Gs) {
    constexpr int KAP = 8 * NA, KBP = 8 * NB, NOUT = KAP * KBP;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    double* s_red = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES + 128);
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(Gs.S, smem, full, empty, s_direct);
        return;
    }
    constexpr int NSET = GramSets<NA, NB>::NSET;
    double acc[NSET][NA][NB][2];
#pragma unroll
    for (int s = 0; s < NSET; ++s)
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[s][i][j][0] = acc[s][i][j][1] = 0.0;
    int it = 0;
    for (int tile = blockIdx.x; tile < Gs.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * Gs.S.T;
        const int nr = (int)((Gs.S.n - r0) < Gs.S.T ? (Gs.S.n - r0) : Gs.S.T);
        if (!s_direct[s]) {
            const unsigned char* st = smem + s * STAGE_BYTES;
            const double* Xt = reinterpret_cast<const double*>(st + Gs.S.off[0]);
            const double* Yt = Gs.same ? Xt : reinterpret_cast<const double*>(st + Gs.S.off[1]);
            gram_tile<NA, NB>(Gs, Xt, Yt, nr, acc);
        } else {
            const double* Xt = Gs.S.p[0] + r0 * Gs.ka;
            const double* Yt = (Gs.same ? Gs.S.p[0] : Gs.S.p[1]) + r0 * Gs.kb;
            gram_tile<NA, NB>(Gs, Xt, Yt, nr, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    // every issued bulk copy has completed (each was waited on), so once all
    // consumer warps are past the loop the ring memory is reused for the combine
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    s_red = reinterpret_cast<double*>(smem);
    const int kq = lane & 3, mg = lane >> 2;
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            double* d = s_red + warp * NOUT + (8 * i + mg) * KBP + 8 * j + 2 * kq;
            double v0 = acc[0][i][j][0], v1 = acc[0][i][j][1];
#pragma unroll
            for (int s = 1; s < NSET; ++s) { v0 += acc[s][i][j][0]; v1 += acc[s][i][j][1]; }   // fixed order
            d[0] = v0;
            d[1] = v1;
        }
    finish_reduce<NOUT>(Gs, s_red, Gs.ka * Gs.kb, Gs.kb, KBP, false);
}

// ka, kb <= 4: FMA consumer (an 8 x 8 DMMA block would waste most lanes).
// Thread t walks rows t, t + NC, ... of each tile; fixed-order shuffle tree per
// warp, then the common CTA / grid reduction.
__global__ void __launch_bounds__(NC + 32, 2) gram_small_stream_kernel(const GramStream Gs) {
    constexpr int NOUT = 16;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(Gs.S, smem, full, empty, s_direct);
        return;
    }
    const int ka = Gs.ka, kb = Gs.kb;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    int it = 0;
    for (int tile = blockIdx.x; tile < Gs.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * Gs.S.T;
        const int nr = (int)((Gs.S.n - r0) < Gs.S.T ? (Gs.S.n - r0) : Gs.S.T);
        const unsigned char* st = smem + s * STAGE_BYTES;
        const bool dir = s_direct[s] != 0;
        const double* Xt = dir ? Gs.S.p[0] + r0 * ka : reinterpret_cast<const double*>(st + Gs.S.off[0]);
        const double* Yt = Gs.same ? Xt : (dir ? Gs.S.p[1] + r0 * kb : reinterpret_cast<const double*>(st + Gs.S.off[1]));
        for (int r = threadIdx.x; r < nr; r += NC) {
            double x[4], y[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) x[a] = a < ka ? Xt[(int64_t)r * ka + a] : 0.0;
#pragma unroll
            for (int b = 0; b < 4; ++b) y[b] = b < kb ? Yt[(int64_t)r * kb + b] : 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    double* s_red = reinterpret_cast<double*>(smem);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            double v = acc[a][b];
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
            if (lane == 0) s_red[warp * NOUT + a * 4 + b] = v;
        }
    finish_reduce<NOUT>(Gs, s_red, ka * kb, kb, 4, false);
}

// coldot: d_c = sum_r X[r,c] Y[r,c], d2_c with Y2 (X, Y, Y2 all k wide)
__global__ void __launch_bounds__(NC + 32, 2) coldot_stream_kernel(const GramStream Gs) {
    constexpr int NOUT = 64;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    double* s_red = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES + 128);
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(Gs.S, smem, full, empty, s_direct);
        return;
    }
    const int k = Gs.ka;
    const bool two = Gs.G2 != nullptr;
    // k | 32: flattened walk over the tile's nr*k elements, thread t always sees
    // column t % k (all lanes busy, conflict-free); otherwise lane = column.
    const bool flat = (32 % k) == 0;
    const int c = flat ? (lane % k) : lane;
    double d1 = 0.0, d2 = 0.0;
    int it = 0;
    for (int tile = blockIdx.x; tile < Gs.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * Gs.S.T;
        const int nr = (int)((Gs.S.n - r0) < Gs.S.T ? (Gs.S.n - r0) : Gs.S.T);
        const unsigned char* st = smem + s * STAGE_BYTES;
        const bool dir = s_direct[s] != 0;
        const double* Xt = dir ? Gs.S.p[0] + r0 * k : reinterpret_cast<const double*>(st + Gs.S.off[0]);
        const double* Yt = Gs.same ? Xt : (dir ? Gs.S.p[1] + r0 * k : reinterpret_cast<const double*>(st + Gs.S.off[1]));
        const double* Y2t = !two ? nullptr
                            : Gs.y2x ? Xt
                                     : (dir ? Gs.S.p[2] + r0 * k : reinterpret_cast<const double*>(st + Gs.S.off[2]));
        if (flat) {
            const int ne = nr * k;
            for (int e = threadIdx.x; e < ne; e += NC) {
                const double x = Xt[e];
                d1 = fma(x, Yt[e], d1);
                if (two) d2 = fma(x, Y2t[e], d2);
            }
        } else if (c < k) {
            for (int r = warp; r < nr; r += NC / 32) {
                const double x = Xt[(int64_t)r * k + c];
                d1 = fma(x, Yt[(int64_t)r * k + c], d1);
                if (two) d2 = fma(x, Y2t[(int64_t)r * k + c], d2);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (flat) {   // lanes l, l + k, l + 2k, ... share a column: fixed xor tree
        for (int m = 16; m >= k; m >>= 1) {
            d1 += __shfl_xor_sync(0xffffffffu, d1, m);
            d2 += __shfl_xor_sync(0xffffffffu, d2, m);
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    s_red = reinterpret_cast<double*>(smem);
    if (!flat || lane < k) {
        s_red[warp * NOUT + lane] = d1;
        s_red[warp * NOUT + 32 + lane] = d2;
    }
    finish_reduce<NOUT>(Gs, s_red, (two ? 2 : 1) * k, k, 32, true);
}

int grid_for(int ntiles, int num_sms) { return ntiles < 2 * num_sms ? ntiles : 2 * num_sms; }

int tile_rows_for(int bytes_per_row) {
    int T = STAGE_BYTES / (bytes_per_row > 0 ? bytes_per_row : 8);
    T &= ~7;  // multiple of 8 rows keeps every full tile 16-byte sized and aligned
    if (T > 1024) T = 1024;
    return T < 8 ? 8 : T;
}

void set_smem(const void* fn, int bytes) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }

template <int NA, int NB>
void gram_stream_t(const GramStream& Gs, int grid, cudaStream_t st) {
    static_assert((NC / 32) * 64 * NA * NB * 8 <= NSTAGE * STAGE_BYTES, "combine buffer must fit in the ring");
    const int smem = NSTAGE * STAGE_BYTES + 128;
    static bool a = false;
    if (!a) { set_smem((const void*)gram_stream_kernel<NA, NB>, smem); a = true; }
    BK_KERNEL(gram_stream_kernel<NA, NB><<<grid, NC + 32, smem, st>>>(Gs));
}

}  // namespace

// ------------------------------------------------------------------ fused block-BiCGStab passes
// Multi-operand Gram on the FP64 tensor cores: G = [X_0 X_1 ..]^T [Y_0 Y_1 ..]
// with every X_i / Y_j one kw-wide stream of the tile (an array read once even
// if it appears in X and Y).  Column c of X is column c % kw of array c / kw.
template <int NA, int NB>
__device__ __forceinline__ void gram_tile_multi(const GramStream& Gs, const double* const (&base)[MAXS], int nr,
                                                double (&acc)[NA][NB][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, mg = lane >> 2;
    const int kw = Gs.kw, ka = Gs.ka, kb = Gs.kb;
    const double* xb[NA];
    const double* yb[NB];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
        const int c = 8 * i + mg;
        xb[i] = c < ka ? base[Gs.xs[c / kw]] + (c % kw) : nullptr;
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        const int c = 8 * j + mg;
        yb[j] = c < kb ? base[Gs.ys[c / kw]] + (c % kw) : nullptr;
    }
    for (int q0 = 4 * warp; q0 < nr; q0 += 4 * (NC / 32)) {
        const int r = q0 + kq;
        const bool rin = r < nr;
        double av[NA], bv[NB];
#pragma unroll
        for (int i = 0; i < NA; ++i) av[i] = (rin && xb[i]) ? xb[i][(int64_t)r * kw] : 0.0;
#pragma unroll
        for (int j = 0; j < NB; ++j) bv[j] = (rin && yb[j]) ? yb[j][(int64_t)r * kw] : 0.0;
#pragma unroll
        for (int i = 0; i < NA; ++i)
#pragma unroll
            for (int j = 0; j < NB; ++j) dmma(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
}

template <int NA, int NB>
__global__ void __launch_bounds__(NC + 32, 2) gram_multi_stream_kernel(const GramStream Gs) {
    constexpr int KAP = 8 * NA, KBP = 8 * NB, NOUT = KAP * KBP + 64;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(Gs.S, smem, full, empty, s_direct);
        return;
    }
    double acc[NA][NB][2];
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // column dots: flattened walk over the tile (kw | 32: thread t sees column t % kw)
    const int kw = Gs.kw;
    double dd[2] = {0.0, 0.0};
    int it = 0;
    for (int tile = blockIdx.x; tile < Gs.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * Gs.S.T;
        const int nr = (int)((Gs.S.n - r0) < Gs.S.T ? (Gs.S.n - r0) : Gs.S.T);
        const unsigned char* st = smem + s * STAGE_BYTES;
        const double* base[MAXS];
#pragma unroll
        for (int q = 0; q < MAXS; ++q)
            base[q] = q < Gs.S.nin ? (s_direct[s] ? Gs.S.p[q] + r0 * Gs.S.w[q]
                                                  : reinterpret_cast<const double*>(st + Gs.S.off[q]))
                                   : nullptr;
        gram_tile_multi<NA, NB>(Gs, base, nr, acc);
        if (Gs.ndot > 0) {
            const int ne = nr * kw;
            const double *a0 = base[Gs.da[0]], *b0 = base[Gs.db[0]];
            const double *a1 = Gs.ndot > 1 ? base[Gs.da[1]] : a0, *b1 = Gs.ndot > 1 ? base[Gs.db[1]] : b0;
            for (int e = threadIdx.x; e < ne; e += NC) {
                dd[0] = fma(a0[e], b0[e], dd[0]);
                dd[1] = fma(a1[e], b1[e], dd[1]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    for (int m = 16; m >= kw; m >>= 1) {   // lanes l, l + kw, ... share a column: fixed xor tree
        dd[0] += __shfl_xor_sync(0xffffffffu, dd[0], m);
        dd[1] += __shfl_xor_sync(0xffffffffu, dd[1], m);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    double* s_red = reinterpret_cast<double*>(smem);
    if (lane < kw) {
        s_red[warp * NOUT + NOUT - 64 + lane] = dd[0];
        s_red[warp * NOUT + NOUT - 32 + lane] = dd[1];
    }
    const int kq = lane & 3, mg = lane >> 2;
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            double* d = s_red + warp * NOUT + (8 * i + mg) * KBP + 8 * j + 2 * kq;
            d[0] = acc[i][j][0];
            d[1] = acc[i][j][1];
        }
    if (finish_reduce<NOUT>(Gs, s_red, Gs.ka * Gs.kb + Gs.ndot * kw, Gs.kb, KBP, false)) small_epilogue(Gs.epi, smem);
}

// Panel Gram: X and Y are lists of 16-column panels.  Lane (mg, kq) loads the
// 16-byte chunk mg (columns 2mg, 2mg+1) of row q0 + kq of each panel with one
// LDS.128 -- 4 rows x 8 chunks = 512 bytes, conflict-free (the 8-byte
// fragment loads of 16-wide rows were 4-way conflicted) -- and the two columns
// feed two PARITY blocks (even / odd columns of the panel) as m8n8k4 DMMA
// fragments; only the output index mapping changes:
// block (2p + e, 2q + f), fragment (m, n) -> G[16p + 2m + e][16q + 2n + f].
template <int NXP, int NYP>
struct PanelSets { static constexpr int NSET = (NXP * NYP <= 1) ? 2 : 1; };

template <int NXP, int NYP>
__global__ void __launch_bounds__(NC + 32, 2) gram_panel_stream_kernel(const GramStream Gs) {
    constexpr int KA = 16 * NXP, KB = 16 * NYP, NOUT = KA * KB + 64;
    constexpr int NSET = PanelSets<NXP, NYP>::NSET;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(Gs.S, smem, full, empty, s_direct);
        return;
    }
    const int kq = lane & 3, mg = lane >> 2;
    double acc[NSET][2 * NXP][2 * NYP][2];
#pragma unroll
    for (int t = 0; t < NSET; ++t)
#pragma unroll
        for (int i = 0; i < 2 * NXP; ++i)
#pragma unroll
            for (int j = 0; j < 2 * NYP; ++j) acc[t][i][j][0] = acc[t][i][j][1] = 0.0;
    const int kw = Gs.kw;
    double dd[2] = {0.0, 0.0};
    int it = 0;
    for (int tile = blockIdx.x; tile < Gs.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * Gs.S.T;
        const int nr = (int)((Gs.S.n - r0) < Gs.S.T ? (Gs.S.n - r0) : Gs.S.T);
        const unsigned char* st = smem + s * STAGE_BYTES;
        const double* base[MAXS];
#pragma unroll
        for (int q = 0; q < MAXS; ++q)
            base[q] = q < Gs.S.nin ? (s_direct[s] ? Gs.S.p[q] + r0 * Gs.S.w[q]
                                                  : reinterpret_cast<const double*>(st + Gs.S.off[q]))
                                   : nullptr;
        const double* xb[NXP];
        const double* yb[NYP];
        int xw[NXP], yw[NYP];
#pragma unroll
        for (int p = 0; p < NXP; ++p) { xb[p] = base[Gs.xps[p]] + Gs.xpo[p] + 2 * mg; xw[p] = Gs.S.w[Gs.xps[p]]; }
#pragma unroll
        for (int p = 0; p < NYP; ++p) { yb[p] = base[Gs.yps[p]] + Gs.ypo[p] + 2 * mg; yw[p] = Gs.S.w[Gs.yps[p]]; }
        // the row loop with the operand loads as a parameter: shared-memory loads (LDS.128)
        // for staged tiles, global loads for the ragged / unaligned ones (generic loads of
        // staged data went through the long-scoreboard path)
        auto rows = [&](auto lda, auto ldb) {
            for (int q0 = 4 * warp; q0 < nr; q0 += 4 * (NC / 32) * NSET) {
                double2 a[NSET][NXP], b[NSET][NYP];
#pragma unroll
                for (int t = 0; t < NSET; ++t) {
                    const int r = q0 + 4 * (NC / 32) * t + kq;
                    const bool rin = r < nr;
#pragma unroll
                    for (int p = 0; p < NXP; ++p) a[t][p] = rin ? lda(p, r) : make_double2(0.0, 0.0);
#pragma unroll
                    for (int p = 0; p < NYP; ++p) b[t][p] = rin ? ldb(p, r) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int t = 0; t < NSET; ++t)
#pragma unroll
                    for (int p = 0; p < NXP; ++p)
#pragma unroll
                        for (int q = 0; q < NYP; ++q) {
                            dmma(acc[t][2 * p][2 * q][0], acc[t][2 * p][2 * q][1], a[t][p].x, b[t][q].x);
                            dmma(acc[t][2 * p][2 * q + 1][0], acc[t][2 * p][2 * q + 1][1], a[t][p].x, b[t][q].y);
                            dmma(acc[t][2 * p + 1][2 * q][0], acc[t][2 * p + 1][2 * q][1], a[t][p].y, b[t][q].x);
                            dmma(acc[t][2 * p + 1][2 * q + 1][0], acc[t][2 * p + 1][2 * q + 1][1], a[t][p].y,
                                 b[t][q].y);
                        }
            }
        };
        const bool dir = s_direct[s] != 0;
        if (!dir) {
            uint32_t xa[NXP], ya[NYP];
#pragma unroll
            for (int p = 0; p < NXP; ++p) xa[p] = smem_u32(xb[p]);
#pragma unroll
            for (int p = 0; p < NYP; ++p) ya[p] = smem_u32(yb[p]);
            rows([&](int p, int r) { return lds_d2(xa[p] + (uint32_t)(r * xw[p]) * 8u); },
                 [&](int p, int r) { return lds_d2(ya[p] + (uint32_t)(r * yw[p]) * 8u); });
        } else {
            rows([&](int p, int r) { return __ldg(reinterpret_cast<const double2*>(xb[p] + (int64_t)r * xw[p])); },
                 [&](int p, int r) { return __ldg(reinterpret_cast<const double2*>(yb[p] + (int64_t)r * yw[p])); });
        }
        if (Gs.ndot > 0) {
            const int ne = nr * kw;
            const double *a0 = base[Gs.da[0]], *b0 = base[Gs.db[0]];
            const double *a1 = Gs.ndot > 1 ? base[Gs.da[1]] : a0, *b1 = Gs.ndot > 1 ? base[Gs.db[1]] : b0;
            if (!dir) {
                const uint32_t sa0 = smem_u32(a0), sb0 = smem_u32(b0), sa1 = smem_u32(a1), sb1 = smem_u32(b1);
                for (int e = threadIdx.x; e < ne; e += NC) {
                    const uint32_t o = (uint32_t)e * 8u;
                    dd[0] = fma(lds_d(sa0 + o), lds_d(sb0 + o), dd[0]);
                    dd[1] = fma(lds_d(sa1 + o), lds_d(sb1 + o), dd[1]);
                }
            } else {
                for (int e = threadIdx.x; e < ne; e += NC) {
                    dd[0] = fma(a0[e], b0[e], dd[0]);
                    dd[1] = fma(a1[e], b1[e], dd[1]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    for (int m = 16; m >= kw; m >>= 1) {
        dd[0] += __shfl_xor_sync(0xffffffffu, dd[0], m);
        dd[1] += __shfl_xor_sync(0xffffffffu, dd[1], m);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    double* s_red = reinterpret_cast<double*>(smem);
    if (lane < kw && kw <= 32) {
        s_red[warp * NOUT + NOUT - 64 + lane] = dd[0];
        s_red[warp * NOUT + NOUT - 32 + lane] = dd[1];
    }
#pragma unroll
    for (int i = 0; i < 2 * NXP; ++i)
#pragma unroll
        for (int j = 0; j < 2 * NYP; ++j) {
            double v0 = acc[0][i][j][0], v1 = acc[0][i][j][1];
#pragma unroll
            for (int t = 1; t < NSET; ++t) { v0 += acc[t][i][j][0]; v1 += acc[t][i][j][1]; }   // fixed order
            const int a = 16 * (i >> 1) + 2 * mg + (i & 1);
            const int b = 16 * (j >> 1) + 4 * kq + (j & 1);
            s_red[warp * NOUT + a * KB + b] = v0;
            s_red[warp * NOUT + a * KB + b + 2] = v1;
        }
    if (finish_reduce<NOUT>(Gs, s_red, Gs.ka * Gs.kb + (Gs.mode == 2 ? Gs.ndot * kw : 0), Gs.kb, KB, false))
        small_epilogue(Gs.epi, smem);
}

// BiCGStab tail, one pass (O6 steps in order):
//   X <- X + P al + w S ;  R <- S - w T ;  P <- R + (P - w V) be ;  rr_c = sum_r R[r,c]^2
// al, be: k x k (B fragments in registers); w = *w_dev.  Streams: 0 X, 1 P, 2 S, 3 T, 4 V.
struct BcgTail {
    Streams S;
    int k;
    const double* al;
    const double* be;
    const double* w_dev;
    double* X;
    double* R;
    double* P;
    const int* halt;
    GramStream red;     // coldot-mode reduction of rr (part, ticket, G = rr)
};

template <int NQ, int NK>
__global__ void __launch_bounds__(NC + 32, 2) bcg_tail_stream_kernel(const BcgTail U) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    if (U.halt && *U.halt) return;
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(U.S, smem, full, empty, s_direct);
        return;
    }
    const int k = U.k, kq = lane & 3, mg = lane >> 2;
    // B fragments of al / be in shared memory, [ks][nb][lane] (conflict-free LDS.64;
    // keeping them in registers spilled at the 96-register cap)
    double* s_ba = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES + 128);
    double* s_bb = s_ba + NQ * NK * 32;
#pragma unroll
    for (int ks = 0; ks < NQ; ++ks)
#pragma unroll
        for (int nb = 0; nb < NK; ++nb) {
            const bool oc = 8 * nb + mg < k;   // (k % 8 == 4: the last block is half padding)
            s_ba[(ks * NK + nb) * 32 + lane] = oc ? U.al[(4 * ks + kq) * k + 8 * nb + mg] : 0.0;
            s_bb[(ks * NK + nb) * 32 + lane] = oc ? U.be[(4 * ks + kq) * k + 8 * nb + mg] : 0.0;
        }
    __syncwarp();
    const double w = *U.w_dev;
    double rr[NK][2];
#pragma unroll
    for (int nb = 0; nb < NK; ++nb) rr[nb][0] = rr[nb][1] = 0.0;
    int it = 0;
    for (int tile = blockIdx.x; tile < U.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * U.S.T;
        const int nr = (int)((U.S.n - r0) < U.S.T ? (U.S.n - r0) : U.S.T);
        const unsigned char* st = smem + s * STAGE_BYTES;
        const double* b[5];
#pragma unroll
        for (int q = 0; q < 5; ++q)
            b[q] = s_direct[s] ? U.S.p[q] + r0 * k : reinterpret_cast<const double*>(st + U.S.off[q]);
        const double *Xt = b[0], *Pt = b[1], *St = b[2], *Tt = b[3], *Vt = b[4];
        for (int rb = 8 * warp; rb < nr; rb += 8 * (NC / 32)) {
            const int r = rb + mg;
            const bool rin = r < nr;
            double ap[NQ], aq[NQ];   // A fragments: P and P - w V (row mg, col 4 ks + kq)
#pragma unroll
            for (int ks = 0; ks < NQ; ++ks) {
                const double p = rin ? Pt[(int64_t)r * k + 4 * ks + kq] : 0.0;
                const double v = rin ? Vt[(int64_t)r * k + 4 * ks + kq] : 0.0;
                ap[ks] = p;
                aq[ks] = fma(-w, v, p);
            }
#pragma unroll
            for (int nb = 0; nb < NK; ++nb) {
                const int c = 8 * nb + 2 * kq;
                const bool cin = rin && c < k;
                double x0 = 0.0, x1 = 0.0, r0v = 0.0, r1v = 0.0;
                if (cin) {
                    const double2 xv = *reinterpret_cast<const double2*>(Xt + (int64_t)r * k + c);
                    const double2 sv = *reinterpret_cast<const double2*>(St + (int64_t)r * k + c);
                    const double2 tv = *reinterpret_cast<const double2*>(Tt + (int64_t)r * k + c);
                    x0 = fma(w, sv.x, xv.x);
                    x1 = fma(w, sv.y, xv.y);
                    r0v = fma(-w, tv.x, sv.x);
                    r1v = fma(-w, tv.y, sv.y);
                }
                double p0 = r0v, p1 = r1v;
#pragma unroll
                for (int ks = 0; ks < NQ; ++ks) {
                    dmma(x0, x1, ap[ks], s_ba[(ks * NK + nb) * 32 + lane]);
                    dmma(p0, p1, aq[ks], s_bb[(ks * NK + nb) * 32 + lane]);
                }
                if (cin) {
                    const int64_t o = (r0 + r) * k + c;
                    *reinterpret_cast<double2*>(U.X + o) = make_double2(x0, x1);
                    *reinterpret_cast<double2*>(U.R + o) = make_double2(r0v, r1v);
                    *reinterpret_cast<double2*>(U.P + o) = make_double2(p0, p1);
                    rr[nb][0] = fma(r0v, r0v, rr[nb][0]);
                    rr[nb][1] = fma(r1v, r1v, rr[nb][1]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    // column sums over the 8 row groups (lanes with equal kq): fixed xor tree
#pragma unroll
    for (int nb = 0; nb < NK; ++nb)
#pragma unroll
        for (int m = 4; m <= 16; m <<= 1) {
            rr[nb][0] += __shfl_xor_sync(0xffffffffu, rr[nb][0], m);
            rr[nb][1] += __shfl_xor_sync(0xffffffffu, rr[nb][1], m);
        }
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    double* s_red = reinterpret_cast<double*>(smem);
    if (mg == 0) {
#pragma unroll
        for (int nb = 0; nb < NK; ++nb) {
            s_red[warp * 64 + 8 * nb + 2 * kq] = rr[nb][0];
            s_red[warp * 64 + 8 * nb + 2 * kq + 1] = rr[nb][1];
        }
    }
    if (finish_reduce<64>(U.red, s_red, k, k, 32, true)) small_epilogue(U.red.epi, smem);
}

// ------------------------------------------------------------------ fused block-CG tail
// X <- X + P al ; R <- R - Q al ; G = R^T R (new R) -- one pass (O4 steps in order).
// Streams: 0 X, 1 P, 2 R, 3 Q.  al: k x k (B fragments in shared memory).  The new R rows
// are written back into the consumed stage tile, and each warp accumulates the Gram of its
// 8-row blocks on the tensor cores; CTA partials + the common fixed-order reduction.
struct CgTail {
    Streams S;
    int k;
    const double* al;
    double* X;
    double* R;
    const int* halt;
    GramStream red;     // gram-mode reduction of G (part, ticket, G, ka = kb = k)
};

template <int NQ, int NK>
__global__ void __launch_bounds__(NC + 32, 2) cg_tail_stream_kernel(const CgTail U) {
    constexpr int KBP = 8 * NK, NOUT = KBP * KBP;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    if (U.halt && *U.halt) return;
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(U.S, smem, full, empty, s_direct);
        return;
    }
    const int k = U.k, kq = lane & 3, mg = lane >> 2;
    double* s_ba = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES + 128);
#pragma unroll
    for (int ks = 0; ks < NQ; ++ks)
#pragma unroll
        for (int nb = 0; nb < NK; ++nb)   // (k % 8 == 4: the last block is half padding)
            s_ba[(ks * NK + nb) * 32 + lane] = 8 * nb + mg < k ? U.al[(4 * ks + kq) * k + 8 * nb + mg] : 0.0;
    __syncwarp();
    double g[NK][NK][2];
#pragma unroll
    for (int i = 0; i < NK; ++i)
#pragma unroll
        for (int j = 0; j < NK; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    int it = 0;
    for (int tile = blockIdx.x; tile < U.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * U.S.T;
        const int nr = (int)((U.S.n - r0) < U.S.T ? (U.S.n - r0) : U.S.T);
        unsigned char* st = smem + s * STAGE_BYTES;
        const bool dir = s_direct[s] != 0;
        const double* Xt = dir ? U.S.p[0] + r0 * k : reinterpret_cast<const double*>(st + U.S.off[0]);
        const double* Pt = dir ? U.S.p[1] + r0 * k : reinterpret_cast<const double*>(st + U.S.off[1]);
        double* Rt = dir ? nullptr : reinterpret_cast<double*>(st + U.S.off[2]);
        const double* Rg = U.S.p[2] + r0 * k;
        const double* Qt = dir ? U.S.p[3] + r0 * k : reinterpret_cast<const double*>(st + U.S.off[3]);
        for (int rb = 8 * warp; rb < nr; rb += 8 * (NC / 32)) {
            const int r = rb + mg;
            const bool rin = r < nr;
            double ap[NQ], aq[NQ];   // A fragments: P and -Q (row mg, col 4 ks + kq)
#pragma unroll
            for (int ks = 0; ks < NQ; ++ks) {
                ap[ks] = rin ? Pt[(int64_t)r * k + 4 * ks + kq] : 0.0;
                aq[ks] = rin ? -Qt[(int64_t)r * k + 4 * ks + kq] : 0.0;
            }
#pragma unroll
            for (int nb = 0; nb < NK; ++nb) {
                const int c = 8 * nb + 2 * kq;
                const bool cin = rin && c < k, cok = c < k;
                double x0 = 0.0, x1 = 0.0, q0 = 0.0, q1 = 0.0;
                if (cin) {
                    const double2 xv = *reinterpret_cast<const double2*>(Xt + (int64_t)r * k + c);
                    const double2 rv = dir ? *reinterpret_cast<const double2*>(Rg + (int64_t)r * k + c)
                                           : *reinterpret_cast<const double2*>(Rt + (int64_t)r * k + c);
                    x0 = xv.x; x1 = xv.y; q0 = rv.x; q1 = rv.y;
                }
#pragma unroll
                for (int ks = 0; ks < NQ; ++ks) {
                    const double b = s_ba[(ks * NK + nb) * 32 + lane];
                    dmma(x0, x1, ap[ks], b);
                    dmma(q0, q1, aq[ks], b);
                }
                if (cin) {
                    const int64_t o = (r0 + r) * k + c;
                    *reinterpret_cast<double2*>(U.X + o) = make_double2(x0, x1);
                    *reinterpret_cast<double2*>(U.R + o) = make_double2(q0, q1);
                }
                if (!dir && cok) *reinterpret_cast<double2*>(Rt + (int64_t)(rb + mg) * k + c) =
                    rin ? make_double2(q0, q1) : make_double2(0.0, 0.0);
            }
            // Gram of the block's new rows (this warp wrote them): two k-steps of 4 rows
            __syncwarp();
            const double* Rn = dir ? U.R + r0 * k : Rt;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr = rb + 4 * h + kq;
                double a[NK];
#pragma unroll
                for (int i = 0; i < NK; ++i) a[i] = (rr < nr && 8 * i + mg < k) ? Rn[(int64_t)rr * k + 8 * i + mg] : 0.0;
#pragma unroll
                for (int i = 0; i < NK; ++i)
#pragma unroll
                    for (int j = 0; j < NK; ++j) dmma(g[i][j][0], g[i][j][1], a[i], a[j]);
            }
            __syncwarp();
        }
        // the new R rows went into the stage with generic stores; the producer's next bulk
        // copy into this stage is an async-proxy write: order them (PTX memory model)
        if (!dir) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    double* s_red = reinterpret_cast<double*>(smem);
#pragma unroll
    for (int i = 0; i < NK; ++i)
#pragma unroll
        for (int j = 0; j < NK; ++j) {
            double* d = s_red + warp * NOUT + (8 * i + mg) * KBP + 8 * j + 2 * kq;
            d[0] = g[i][j][0];
            d[1] = g[i][j][1];
        }
    if (finish_reduce<NOUT>(U.red, s_red, k * k, k, KBP, false)) small_epilogue(U.red.epi, smem);
}

// ------------------------------------------------------------------ single-reduction block-CG tail
// O11 (oracle block_cg1), one pass:  P <- R + P be ;  Q <- W + Q be ;  X <- X + P al ;  R <- R - Q al
// (new P, Q).  Streams: 0 X, 1 R, 2 P, 3 W, 4 Q.  al, be: k x k (B fragments in shared memory).
// Each warp owns 8-row blocks: the new P / Q rows are written back into the consumed stage
// tile and re-read as A fragments of the X / R updates by the same warp.  No reduction: the
// iteration's one reduction pass is the next W = A R apply (RED 4).
struct Cg1Tail {
    Streams S;
    int k;
    const double* al;
    const double* be;
    double* X;
    double* R;
    double* P;
    double* Q;
    const int* halt;
};

template <int NQ, int NK>
__global__ void __launch_bounds__(NC + 32, 2) cg1_tail_stream_kernel(const Cg1Tail U) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    int* s_direct = reinterpret_cast<int*>(empty + NSTAGE);
    if (U.halt && *U.halt) return;
    stream_setup(full, empty);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NC / 32) {
        if (lane == 0) stream_produce(U.S, smem, full, empty, s_direct);
        return;
    }
    const int k = U.k, kq = lane & 3, mg = lane >> 2;
    double* s_ba = reinterpret_cast<double*>(smem + NSTAGE * STAGE_BYTES + 128);
    double* s_bb = s_ba + NQ * NK * 32;
#pragma unroll
    for (int ks = 0; ks < NQ; ++ks)
#pragma unroll
        for (int nb = 0; nb < NK; ++nb) {   // (k % 8 == 4: the last block is half padding)
            const bool oc = 8 * nb + mg < k;
            s_ba[(ks * NK + nb) * 32 + lane] = oc ? U.al[(4 * ks + kq) * k + 8 * nb + mg] : 0.0;
            s_bb[(ks * NK + nb) * 32 + lane] = oc ? U.be[(4 * ks + kq) * k + 8 * nb + mg] : 0.0;
        }
    __syncwarp();
    int it = 0;
    for (int tile = blockIdx.x; tile < U.S.ntiles; tile += gridDim.x, ++it) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int64_t r0 = (int64_t)tile * U.S.T;
        const int nr = (int)((U.S.n - r0) < U.S.T ? (U.S.n - r0) : U.S.T);
        unsigned char* st = smem + s * STAGE_BYTES;
        const bool dir = s_direct[s] != 0;
        const double* Xt = dir ? U.S.p[0] + r0 * k : reinterpret_cast<const double*>(st + U.S.off[0]);
        const double* Rt = dir ? U.S.p[1] + r0 * k : reinterpret_cast<const double*>(st + U.S.off[1]);
        // direct tiles: the new P / Q rows are re-read from global memory (this warp wrote them)
        double* Pt = dir ? U.P + r0 * k : reinterpret_cast<double*>(st + U.S.off[2]);
        const double* Wt = dir ? U.S.p[3] + r0 * k : reinterpret_cast<const double*>(st + U.S.off[3]);
        double* Qt = dir ? U.Q + r0 * k : reinterpret_cast<double*>(st + U.S.off[4]);
        for (int rb = 8 * warp; rb < nr; rb += 8 * (NC / 32)) {
            const int r = rb + mg;
            const bool rin = r < nr;
            double ap[NQ], aq[NQ];   // A fragments of the old P, Q (row mg, col 4 ks + kq)
#pragma unroll
            for (int ks = 0; ks < NQ; ++ks) {
                ap[ks] = rin ? Pt[(int64_t)r * k + 4 * ks + kq] : 0.0;
                aq[ks] = rin ? Qt[(int64_t)r * k + 4 * ks + kq] : 0.0;
            }
            __syncwarp();   // every lane holds its old P / Q fragments before the rows are overwritten
#pragma unroll
            for (int nb = 0; nb < NK; ++nb) {
                const int c = 8 * nb + 2 * kq;
                const bool cin = rin && c < k;
                double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
                if (cin) {
                    const double2 rv = *reinterpret_cast<const double2*>(Rt + (int64_t)r * k + c);
                    const double2 wv = *reinterpret_cast<const double2*>(Wt + (int64_t)r * k + c);
                    p0 = rv.x; p1 = rv.y; q0 = wv.x; q1 = wv.y;
                }
#pragma unroll
                for (int ks = 0; ks < NQ; ++ks) {
                    const double b = s_bb[(ks * NK + nb) * 32 + lane];
                    dmma(p0, p1, ap[ks], b);
                    dmma(q0, q1, aq[ks], b);
                }
                if (cin) {
                    const int64_t o = (r0 + r) * k + c;
                    if (!dir) {
                        *reinterpret_cast<double2*>(U.P + o) = make_double2(p0, p1);
                        *reinterpret_cast<double2*>(U.Q + o) = make_double2(q0, q1);
                    }
                    *reinterpret_cast<double2*>(Pt + (int64_t)r * k + c) = make_double2(p0, p1);
                    *reinterpret_cast<double2*>(Qt + (int64_t)r * k + c) = make_double2(q0, q1);
                }
            }
            __syncwarp();   // the block's new P / Q rows are visible to the whole warp
            double bp[NQ], bq[NQ];   // A fragments of the new P and of -(new Q)
#pragma unroll
            for (int ks = 0; ks < NQ; ++ks) {
                bp[ks] = rin ? Pt[(int64_t)r * k + 4 * ks + kq] : 0.0;
                bq[ks] = rin ? -Qt[(int64_t)r * k + 4 * ks + kq] : 0.0;
            }
#pragma unroll
            for (int nb = 0; nb < NK; ++nb) {
                const int c = 8 * nb + 2 * kq;
                const bool cin = rin && c < k;
                double x0 = 0.0, x1 = 0.0, v0 = 0.0, v1 = 0.0;
                if (cin) {
                    const double2 xv = *reinterpret_cast<const double2*>(Xt + (int64_t)r * k + c);
                    const double2 rv = *reinterpret_cast<const double2*>(Rt + (int64_t)r * k + c);
                    x0 = xv.x; x1 = xv.y; v0 = rv.x; v1 = rv.y;
                }
#pragma unroll
                for (int ks = 0; ks < NQ; ++ks) {
                    const double b = s_ba[(ks * NK + nb) * 32 + lane];
                    dmma(x0, x1, bp[ks], b);
                    dmma(v0, v1, bq[ks], b);
                }
                if (cin) {
                    const int64_t o = (r0 + r) * k + c;
                    *reinterpret_cast<double2*>(U.X + o) = make_double2(x0, x1);
                    *reinterpret_cast<double2*>(U.R + o) = make_double2(v0, v1);
                }
            }
            __syncwarp();
        }
        // generic stores went into the stage; the producer's next bulk copy into it is an
        // async-proxy write: order them (PTX memory model)
        if (!dir) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

int panel_mode() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("BK_GRAM_PANEL");
        v = e ? atoi(e) : 1;
    }
    return v;
}
bool panel_enabled() { return panel_mode() != 0; }

bool launch_panel(const GramStream& Gs, int grid, cudaStream_t st) {
    const int smem = NSTAGE * STAGE_BYTES + 128;
#define BK_GP(A, B)                                                                              \
    if (Gs.nxp == A && Gs.nyp == B) {                                                            \
        static_assert((NC / 32) * (256 * A * B + 64) * 8 <= NSTAGE * STAGE_BYTES, "combine");    \
        static bool at = false;                                                                  \
        if (!at) { set_smem((const void*)gram_panel_stream_kernel<A, B>, smem); at = true; }     \
        BK_KERNEL(gram_panel_stream_kernel<A, B><<<grid, NC + 32, smem, st>>>(Gs));               \
        return true;                                                                             \
    }
    BK_GP(1, 1) BK_GP(1, 2) BK_GP(2, 1) BK_GP(2, 2) BK_GP(3, 1)
#undef BK_GP
    return false;
}

// ------------------------------------------------------------------ launchers (return false = not applicable)
// CTA partials + group partials (<= 32 groups of 16), NOUT <= 2048 each
size_t stream_part_doubles(int num_sms) { return (size_t)(2 * num_sms + 40) * 2048; }

static void stream_geom(Streams& S, int nin, int64_t n);

bool launch_update_stream(const UpdArgs& u, int num_sms, cudaStream_t st) {
    // contiguous operands only, kp and k <= 32, out not aliasing P/Xin/W rows in other tiles is fine
    // (a strided output -- e.g. a GMRES basis block -- is written row by row from registers)
    if (u.kp < 0 || u.kp > 32 || u.k > 32 || (u.kp > 0 && u.ldp != u.kp) || u.ldo < u.k) return false;
    if (u.ldo != u.k && ((u.ldo & 1) || u.k % 2)) return false;
    // in place (out == P, e.g. block CG's P = R + P be): the DMMA kernel reads a row's P fragments
    // (from the stage, or -- direct tiles -- from global memory before a __syncwarp) before any
    // lane writes it; the FMA kernel does not, so it leaves in-place updates to blas.cu
    if (u.kp > 0 && (const double*)u.out == u.P &&
        !(u.ldo == u.kp && u.kp == u.k && u.k % 4 == 0 && (!getenv("BK_UPD") || strcmp(getenv("BK_UPD"), "fma") != 0)))
        return false;
    if (u.a != 0.0 && (u.ldxin != u.k || !u.Xin)) return false;
    if (u.W && u.ldw != u.k) return false;
    if (u.kp == 0 && u.a == 0.0 && !u.W) return false;
    if (((uintptr_t)u.out & 15) || (u.kp > 0 && ((uintptr_t)u.P & 15))) return false;
    const int cw = (u.k % 4 == 0) ? 4 : ((u.k % 2 == 0) ? 2 : 1);
    UpdStream U{};
    int nin = 0;
    U.iP = -1;
    if (u.kp > 0) { U.iP = nin; U.S.p[nin] = u.P; U.S.w[nin] = u.kp; ++nin; }
    U.iX = -1; U.iW = -1;
    if (u.a != 0.0) { U.iX = nin; U.S.p[nin] = u.Xin; U.S.w[nin] = u.k; ++nin; }
    if (u.W) { U.iW = nin; U.S.p[nin] = u.W; U.S.w[nin] = u.k; ++nin; }
    int bpr = 0;
    for (int j = 0; j < nin; ++j) bpr += U.S.w[j] * 8;
    U.S.nin = nin;
    U.S.T = tile_rows_for(bpr);
    int off = 0;
    for (int j = 0; j < nin; ++j) { U.S.off[j] = off; off += U.S.T * U.S.w[j] * 8; off = (off + 127) & ~127; }
    if (off > STAGE_BYTES) { U.S.T /= 2; U.S.T &= ~7; off = 0;
        for (int j = 0; j < nin; ++j) { U.S.off[j] = off; off += U.S.T * U.S.w[j] * 8; off = (off + 127) & ~127; } }
    U.S.n = u.n;
    U.S.ntiles = (int)((u.n + U.S.T - 1) / U.S.T);
    U.kp = u.kp; U.k = u.k; U.cw = cw;
    U.a = u.a; U.s = u.s; U.w_host = u.w_host; U.w_dev = u.w_dev;
    U.C = u.C; U.out = u.out; U.ldo = u.ldo; U.halt = u.halt;
    const int smem = NSTAGE * STAGE_BYTES + 128 + 32 * 32 * 8;
    const int grid = grid_for(U.S.ntiles, num_sms);
    if (grid <= 0) return true;
    static int mma = -1;
    if (mma < 0) {
        const char* e = getenv("BK_UPD");
        mma = (e && strcmp(e, "fma") == 0) ? 0 : 1;
    }
    if (mma && u.kp > 0 && u.k % 4 == 0 && u.kp % 4 == 0) {   // (k = 12, 20, 28: padded last block)
        const int nq = u.kp / 4, nk = (u.k + 7) / 8;
#define BK_UM(Q, K)                                                                            \
    if (nq == Q && nk == K) {                                                                  \
        static bool at = false;                                                                \
        if (!at) { set_smem((const void*)upd_stream_mma_kernel<Q, K>, smem); at = true; }       \
        BK_KERNEL(upd_stream_mma_kernel<Q, K><<<grid, NC + 32, smem, st>>>(U));                 \
        return true;                                                                           \
    }
        BK_UM(1, 1) BK_UM(2, 1) BK_UM(3, 1) BK_UM(4, 1) BK_UM(5, 1) BK_UM(6, 1) BK_UM(7, 1) BK_UM(8, 1)
        BK_UM(1, 2) BK_UM(2, 2) BK_UM(3, 2) BK_UM(4, 2) BK_UM(5, 2) BK_UM(6, 2) BK_UM(7, 2) BK_UM(8, 2)
        BK_UM(1, 3) BK_UM(2, 3) BK_UM(3, 3) BK_UM(4, 3) BK_UM(5, 3) BK_UM(6, 3) BK_UM(7, 3) BK_UM(8, 3)
        BK_UM(1, 4) BK_UM(2, 4) BK_UM(3, 4) BK_UM(4, 4) BK_UM(5, 4) BK_UM(6, 4) BK_UM(7, 4) BK_UM(8, 4)
#undef BK_UM
    }
    static bool a1 = false, a2 = false, a4 = false;
    if (cw == 4) {
        if (!a4) { set_smem((const void*)upd_stream_kernel<4>, smem); a4 = true; }
        BK_KERNEL(upd_stream_kernel<4><<<grid, NC + 32, smem, st>>>(U));
    } else if (cw == 2) {
        if (!a2) { set_smem((const void*)upd_stream_kernel<2>, smem); a2 = true; }
        BK_KERNEL(upd_stream_kernel<2><<<grid, NC + 32, smem, st>>>(U));
    } else {
        if (!a1) { set_smem((const void*)upd_stream_kernel<1>, smem); a1 = true; }
        BK_KERNEL(upd_stream_kernel<1><<<grid, NC + 32, smem, st>>>(U));
    }
    return true;
}

bool launch_gram_stream(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                        double* G, double* part, int* ticket, int num_sms, cudaStream_t st) {
    if (ka > 32 || kb > 32 || ldx != ka || ldy != kb || n <= 0) return false;
    if (((uintptr_t)X & 15) || ((uintptr_t)Y & 15)) return false;
    GramStream Gs{};
    Gs.same = (X == Y && ka == kb) ? 1 : 0;
    int nin = 0;
    Gs.S.p[nin] = X; Gs.S.w[nin] = ka; ++nin;
    if (!Gs.same) { Gs.S.p[nin] = Y; Gs.S.w[nin] = kb; ++nin; }
    int bpr = 0;
    for (int j = 0; j < nin; ++j) bpr += Gs.S.w[j] * 8;
    Gs.S.nin = nin;
    Gs.S.T = tile_rows_for(bpr);
    int off = 0;
    for (int j = 0; j < nin; ++j) { Gs.S.off[j] = off; off += Gs.S.T * Gs.S.w[j] * 8; off = (off + 127) & ~127; }
    if (off > STAGE_BYTES) { Gs.S.T /= 2; Gs.S.T &= ~7; off = 0;
        for (int j = 0; j < nin; ++j) { Gs.S.off[j] = off; off += Gs.S.T * Gs.S.w[j] * 8; off = (off + 127) & ~127; } }
    Gs.S.n = n;
    Gs.S.ntiles = (int)((n + Gs.S.T - 1) / Gs.S.T);
    Gs.ka = ka; Gs.kb = kb; Gs.part = part; Gs.ticket = ticket; Gs.G = G; Gs.G2 = nullptr;
    const int grid = grid_for(Gs.S.ntiles, num_sms);
    // (measured: the 8-byte fragment kernel is faster for the plain Gram once it does not
    // spill -- k = 16: 49 vs 52 us, k = 32: 96 vs 113 us; BK_GRAM_PANEL=2 forces panels)
    if (ka % 16 == 0 && kb % 16 == 0 && panel_mode() == 2) {
        Gs.kw = 16;
        Gs.nxp = ka / 16; Gs.nyp = kb / 16;
        for (int p = 0; p < Gs.nxp; ++p) { Gs.xps[p] = 0; Gs.xpo[p] = 16 * p; }
        for (int p = 0; p < Gs.nyp; ++p) { Gs.yps[p] = Gs.same ? 0 : 1; Gs.ypo[p] = 16 * p; }
        if (launch_panel(Gs, grid, st)) return true;
    }
    if (ka <= 4 && kb <= 4) {
        const int smem = NSTAGE * STAGE_BYTES + 128;
        static bool a = false;
        if (!a) { set_smem((const void*)gram_small_stream_kernel, smem); a = true; }
        BK_KERNEL(gram_small_stream_kernel<<<grid, NC + 32, smem, st>>>(Gs));
        return true;
    }
    const int na = (ka + 7) / 8, nb = (kb + 7) / 8;
#define BK_GS(A, B) if (na == A && nb == B) { gram_stream_t<A, B>(Gs, grid, st); return true; }
    BK_GS(1, 1) BK_GS(1, 2) BK_GS(1, 3) BK_GS(1, 4) BK_GS(2, 1) BK_GS(2, 2) BK_GS(2, 3) BK_GS(2, 4)
    BK_GS(3, 1) BK_GS(3, 2) BK_GS(3, 3) BK_GS(3, 4) BK_GS(4, 1) BK_GS(4, 2) BK_GS(4, 3) BK_GS(4, 4)
#undef BK_GS
    return false;
}

bool launch_coldot_stream(int64_t n, int k, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                          const double* Y2, int64_t ldy2, double* d, double* d2, double* part, int* ticket,
                          int num_sms, cudaStream_t st) {
    if (k > 32 || ldx != k || ldy != k || (Y2 && ldy2 != k) || n <= 0) return false;
    if (((uintptr_t)X & 15) || ((uintptr_t)Y & 15) || (Y2 && ((uintptr_t)Y2 & 15))) return false;
    GramStream Gs{};
    Gs.same = (X == Y) ? 1 : 0;
    int nin = 0;
    Gs.S.p[nin] = X; Gs.S.w[nin] = k; ++nin;
    Gs.S.p[nin] = Gs.same ? X : Y; Gs.S.w[nin] = Gs.same ? 0 : k; if (!Gs.same) ++nin; else Gs.S.p[1] = X;
    if (Y2) {
        if (Gs.same) { Gs.S.p[1] = X; Gs.S.w[1] = 0; }
        Gs.y2x = (Y2 == X) ? 1 : 0;   // <T,S>, <T,T>: T streamed once
        Gs.S.p[2] = Y2; Gs.S.w[2] = Gs.y2x ? 0 : k;
        nin = 3;
    }
    // compact: stream list may contain a zero-width slot (same == 1) -- it moves no bytes
    int bpr = 0;
    for (int j = 0; j < nin; ++j) bpr += Gs.S.w[j] * 8;
    Gs.S.nin = nin;
    Gs.S.T = tile_rows_for(bpr);
    int off = 0;
    for (int j = 0; j < nin; ++j) { Gs.S.off[j] = off; off += Gs.S.T * Gs.S.w[j] * 8; off = (off + 127) & ~127; }
    if (off > STAGE_BYTES) { Gs.S.T /= 2; Gs.S.T &= ~7; off = 0;
        for (int j = 0; j < nin; ++j) { Gs.S.off[j] = off; off += Gs.S.T * Gs.S.w[j] * 8; off = (off + 127) & ~127; } }
    Gs.S.n = n;
    Gs.S.ntiles = (int)((n + Gs.S.T - 1) / Gs.S.T);
    Gs.ka = k; Gs.kb = k; Gs.part = part; Gs.ticket = ticket; Gs.G = d; Gs.G2 = Y2 ? d2 : nullptr;
    const int grid = grid_for(Gs.S.ntiles, num_sms);
    const int smem = NSTAGE * STAGE_BYTES + 128;
    static bool a = false;
    if (!a) { set_smem((const void*)coldot_stream_kernel, smem); a = true; }
    BK_KERNEL(coldot_stream_kernel<<<grid, NC + 32, smem, st>>>(Gs));
    return true;
}

// Stream geometry shared by the fused launchers: nin operands of width w each.
static void stream_geom(Streams& S, int nin, int64_t n) {
    int bpr = 0;
    for (int j = 0; j < nin; ++j) bpr += S.w[j] * 8;
    S.nin = nin;
    S.T = tile_rows_for(bpr);
    auto lay = [&]() {
        int off = 0;
        for (int j = 0; j < nin; ++j) { S.off[j] = off; off += S.T * S.w[j] * 8; off = (off + 127) & ~127; }
        return off;
    };
    while (lay() > STAGE_BYTES && S.T > 8) S.T = (S.T / 2) & ~7;
    S.n = n;
    S.ntiles = (int)((n + S.T - 1) / S.T);
}

bool launch_gram_multi_stream(int64_t n, int kw, int nxa, const int* xs, int nya, const int* ys, int nin,
                              const double* const* arrays, double* const (*blk)[2], double* part, int* ticket,
                              int num_sms, cudaStream_t st, int ndot, const int (*dpair)[2], double* const* dots,
                              const SmallEpi* epi) {
    if (kw < 1 || kw > 16 || n <= 0 || nin < 1 || nin > MAXS || nxa < 1 || nxa > 3 || nya < 1 || nya > 2) return false;
    if (ndot < 0 || ndot > 2 || (ndot > 0 && 32 % kw != 0)) return false;
    GramStream Gs{};
    for (int q = 0; q < nin; ++q) {
        if ((uintptr_t)arrays[q] & 15) return false;
        Gs.S.p[q] = arrays[q];
        Gs.S.w[q] = kw;
    }
    stream_geom(Gs.S, nin, n);
    Gs.mode = 2; Gs.kw = kw; Gs.nxa = nxa; Gs.nya = nya;
    for (int i = 0; i < nxa; ++i) Gs.xs[i] = xs[i];
    for (int j = 0; j < nya; ++j) Gs.ys[j] = ys[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 2; ++j) Gs.blk[i][j] = (i < nxa && j < nya) ? blk[i][j] : nullptr;
    Gs.ka = nxa * kw; Gs.kb = nya * kw; Gs.part = part; Gs.ticket = ticket;
    Gs.ndot = ndot;
    for (int q = 0; q < ndot; ++q) { Gs.da[q] = dpair[q][0]; Gs.db[q] = dpair[q][1]; Gs.dots[q] = dots[q]; }
    if (epi) Gs.epi = *epi;
    const int grid = grid_for(Gs.S.ntiles, num_sms);
    if (kw == 16 && panel_enabled()) {   // conflict-free 16-byte fragment loads (parity blocks)
        Gs.nxp = nxa; Gs.nyp = nya;
        for (int i = 0; i < nxa; ++i) { Gs.xps[i] = xs[i]; Gs.xpo[i] = 0; }
        for (int j = 0; j < nya; ++j) { Gs.yps[j] = ys[j]; Gs.ypo[j] = 0; }
        if (launch_panel(Gs, grid, st)) return true;
    }
    const int na = (Gs.ka + 7) / 8, nb = (Gs.kb + 7) / 8;
    const int smem = NSTAGE * STAGE_BYTES + 128;
#define BK_GM(A, B)                                                                              \
    if (na == A && nb == B) {                                                                    \
        static_assert((NC / 32) * (64 * A * B + 64) * 8 <= NSTAGE * STAGE_BYTES, "combine buffer"); \
        static bool at = false;                                                                  \
        if (!at) { set_smem((const void*)gram_multi_stream_kernel<A, B>, smem); at = true; }     \
        BK_KERNEL(gram_multi_stream_kernel<A, B><<<grid, NC + 32, smem, st>>>(Gs));               \
        return true;                                                                             \
    }
    // kw <= 8: (1..3) x (1..2) blocks of 8; kw = 16: (2..6) x (2..4)
    BK_GM(1, 1) BK_GM(1, 2) BK_GM(2, 1) BK_GM(3, 1) BK_GM(2, 2) BK_GM(3, 2) BK_GM(2, 3)
    BK_GM(2, 4) BK_GM(4, 2) BK_GM(6, 2) BK_GM(4, 4)
#undef BK_GM
    return false;
}

bool launch_bcg_tail_stream(int64_t n, int k, double* X, double* R, double* P, const double* S, const double* T,
                            const double* V, const double* al, const double* be, const double* w_dev, double* rr,
                            const int* halt, double* part, int* ticket, int num_sms, cudaStream_t st,
                            const SmallEpi* epi, const double* Pin) {
    if (n <= 0 || k % 4 != 0 || k > 32) return false;
    const double* arr[5] = {X, Pin ? Pin : P, S, T, V};
    BcgTail U{};
    for (int q = 0; q < 5; ++q) {
        if ((uintptr_t)arr[q] & 15) return false;
        U.S.p[q] = arr[q];
        U.S.w[q] = k;
    }
    if ((uintptr_t)R & 15) return false;
    stream_geom(U.S, 5, n);
    U.k = k; U.al = al; U.be = be; U.w_dev = w_dev; U.X = X; U.R = R; U.P = P; U.halt = halt;
    U.red.part = part; U.red.ticket = ticket; U.red.G = rr; U.red.G2 = nullptr;
    if (epi) U.red.epi = *epi;
    const int grid = grid_for(U.S.ntiles, num_sms);
    const int nq = k / 4, nk = (k + 7) / 8;
    const int smem = NSTAGE * STAGE_BYTES + 128 + 2 * nq * nk * 32 * 8;
#define BK_BT(Q, K)                                                                              \
    if (nq == Q && nk == K) {                                                                    \
        static bool at = false;                                                                  \
        if (!at) { set_smem((const void*)bcg_tail_stream_kernel<Q, K>, smem); at = true; }       \
        BK_KERNEL(bcg_tail_stream_kernel<Q, K><<<grid, NC + 32, smem, st>>>(U));                  \
        return true;                                                                             \
    }
    BK_BT(1, 1) BK_BT(2, 1) BK_BT(3, 2) BK_BT(4, 2) BK_BT(6, 3) BK_BT(8, 4)
#undef BK_BT
    return false;
}

bool launch_cg_tail_stream(int64_t n, int k, double* X, double* R, const double* P, const double* Q,
                           const double* al, double* G, const int* halt, double* part, int* ticket, int num_sms,
                           cudaStream_t st, const SmallEpi* epi, const double* Rin) {
    if (n <= 0 || k % 4 != 0 || k > 32) return false;
    const double* arr[4] = {X, P, Rin ? Rin : R, Q};
    CgTail U{};
    for (int q = 0; q < 4; ++q) {
        if ((uintptr_t)arr[q] & 15) return false;
        U.S.p[q] = arr[q];
        U.S.w[q] = k;
    }
    stream_geom(U.S, 4, n);
    U.k = k; U.al = al; U.X = X; U.R = R; U.halt = halt;
    U.red.part = part; U.red.ticket = ticket; U.red.G = G; U.red.G2 = nullptr; U.red.ka = k; U.red.kb = k;
    if (epi) U.red.epi = *epi;
    const int grid = grid_for(U.S.ntiles, num_sms);
    const int nq = k / 4, nk = (k + 7) / 8;
    const int smem = NSTAGE * STAGE_BYTES + 128 + nq * nk * 32 * 8;
#define BK_CT(Q, K)                                                                              \
    if (nq == Q && nk == K) {                                                                    \
        static bool at = false;                                                                  \
        if (!at) { set_smem((const void*)cg_tail_stream_kernel<Q, K>, smem); at = true; }        \
        BK_KERNEL(cg_tail_stream_kernel<Q, K><<<grid, NC + 32, smem, st>>>(U));                   \
        return true;                                                                             \
    }
    BK_CT(1, 1) BK_CT(2, 1) BK_CT(3, 2) BK_CT(4, 2) BK_CT(6, 3) BK_CT(8, 4)
#undef BK_CT
    return false;
}

bool launch_cg1_tail_stream(int64_t n, int k, double* X, double* R, double* P, const double* W, double* Q,
                            const double* al, const double* be, const int* halt, int num_sms, cudaStream_t st,
                            const double* Rin) {
    if (n <= 0 || k % 4 != 0 || k > 16) return false;
    const double* arr[5] = {X, Rin ? Rin : R, P, W, Q};
    Cg1Tail U{};
    for (int q = 0; q < 5; ++q) {
        if ((uintptr_t)arr[q] & 15) return false;
        U.S.p[q] = arr[q];
        U.S.w[q] = k;
    }
    stream_geom(U.S, 5, n);
    U.k = k; U.al = al; U.be = be; U.X = X; U.R = R; U.P = P; U.Q = Q; U.halt = halt;
    const int grid = grid_for(U.S.ntiles, num_sms);
    const int nq = k / 4, nk = (k + 7) / 8;
    const int smem = NSTAGE * STAGE_BYTES + 128 + 2 * nq * nk * 32 * 8;
#define BK_C1(Q_, K_)                                                                            \
    if (nq == Q_ && nk == K_) {                                                                  \
        static bool at = false;                                                                  \
        if (!at) { set_smem((const void*)cg1_tail_stream_kernel<Q_, K_>, smem); at = true; }     \
        BK_KERNEL(cg1_tail_stream_kernel<Q_, K_><<<grid, NC + 32, smem, st>>>(U));                \
        return true;                                                                             \
    }
    BK_C1(1, 1) BK_C1(2, 1) BK_C1(3, 2) BK_C1(4, 2)
#undef BK_C1
    return false;
}

}  // namespace bk
