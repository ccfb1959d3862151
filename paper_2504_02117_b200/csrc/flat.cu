// flat.cu -- narrow (k <= 4) Gram and update passes without the TMA ring.
//
// At k <= 4 a row of each operand is 8-32 bytes, so a plain grid-stride loop with several
// independent rows per thread keeps enough loads in flight, and the fixed cost of the
// persistent TMA-ring kernels (stage setup, one producer thread per CTA, two-level ticket
// tree) dominated them: on c2 the k = 1 Gram moved 16.8 MB in 16.4 us (0.16 of HBM) and the
// k = 1 update 25 MB in 13.8 us.  These kernels are what the small-k
// DIRK baseline (k = 1 sequential stepping) and Algorithm 1's narrow windows run.
//
//   gram_flat_kernel   G = X^T Y (ka, kb <= 4, contiguous rows): per-thread accumulators,
//                      fixed xor-shuffle tree per warp, fixed warp order per block, one
//                      block partial each, and the LAST block (one ticket) sums the partials
//                      in a fixed order -- bitwise reproducible, no atomics on data.
//   upd_flat_kernel    out = a Xin + s P C + w W (k, kp <= 4, contiguous rows), C in registers.
#include "bk_internal.h"

namespace bk {
namespace {

constexpr int FT = 512;       // threads per block
constexpr int FU = 4;         // rows per thread per loop trip (independent loads in flight)

template <int W>
__device__ __forceinline__ void load_row(const double* __restrict__ p, double (&v)[4]) {
    if constexpr (W == 4) {
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
    } else if constexpr (W == 2) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    } else {
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = __ldg(p + j);
    }
}

template <int KA, int KB>
__global__ void __launch_bounds__(FT) gram_flat_kernel(int64_t n, const double* __restrict__ X,
                                                       const double* __restrict__ Y, double* __restrict__ G,
                                                       double* __restrict__ part, int* __restrict__ ticket) {
    constexpr int NO = KA * KB;
    double acc[KA][KB];
#pragma unroll
    for (int a = 0; a < KA; ++a)
#pragma unroll
        for (int b = 0; b < KB; ++b) acc[a][b] = 0.0;
    const int64_t S = (int64_t)gridDim.x * FT;
    for (int64_t r0 = (int64_t)blockIdx.x * FT + threadIdx.x; r0 < n; r0 += FU * S) {
        double x[FU][4], y[FU][4];
#pragma unroll
        for (int u = 0; u < FU; ++u) {
            const int64_t r = r0 + u * S;
#pragma unroll
            for (int j = 0; j < 4; ++j) x[u][j] = y[u][j] = 0.0;
            if (r < n) {
                load_row<KA>(X + r * KA, x[u]);
                load_row<KB>(Y + r * KB, y[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < FU; ++u)
#pragma unroll
            for (int a = 0; a < KA; ++a)
#pragma unroll
                for (int b = 0; b < KB; ++b) acc[a][b] = fma(x[u][a], y[u][b], acc[a][b]);
    }
    __shared__ double s_w[FT / 32][NO];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < KA; ++a)
#pragma unroll
        for (int b = 0; b < KB; ++b) {
            double v = acc[a][b];
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
            if (lane == 0) s_w[warp][a * KB + b] = v;
        }
    __syncthreads();
    if (threadIdx.x < NO) {
        double v = s_w[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < FT / 32; ++w) v += s_w[w][threadIdx.x];
        part[(int64_t)blockIdx.x * NO + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last block: thread t sums partial rows t, t + FT, ... (every output at once: one batch of
    // independent loads), then the same fixed shuffle / warp-order tree as above
    double f[NO];
#pragma unroll
    for (int q = 0; q < NO; ++q) f[q] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += FT)
#pragma unroll
        for (int q = 0; q < NO; ++q) f[q] += __ldcg(part + (int64_t)b * NO + q);
    __syncthreads();   // s_w reused
#pragma unroll
    for (int q = 0; q < NO; ++q) {
        double v = f[q];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) s_w[warp][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < NO) {
        double v = s_w[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < FT / 32; ++w) v += s_w[w][threadIdx.x];
        G[threadIdx.x] = v;
    }
    if (threadIdx.x == 0) *ticket = 0;
}

template <int K, int KP>
__global__ void __launch_bounds__(FT) upd_flat_kernel(const UpdArgs u) {
    if (u.halt && *u.halt) return;
    double c[KP > 0 ? KP : 1][K];
#pragma unroll
    for (int q = 0; q < (KP > 0 ? KP : 1); ++q)
#pragma unroll
        for (int j = 0; j < K; ++j) c[q][j] = KP > 0 ? u.C[q * K + j] : 0.0;
    const double wv = u.W ? (u.w_dev ? u.w_host * *u.w_dev : u.w_host) : 0.0;
    const bool hx = u.a != 0.0 && u.Xin;
    const int64_t S = (int64_t)gridDim.x * FT, n = u.n;
    for (int64_t r0 = (int64_t)blockIdx.x * FT + threadIdx.x; r0 < n; r0 += FU * S) {
        double p[FU][4], x[FU][4], w[FU][4];
#pragma unroll
        for (int t = 0; t < FU; ++t) {
            const int64_t r = r0 + t * S;
#pragma unroll
            for (int j = 0; j < 4; ++j) p[t][j] = x[t][j] = w[t][j] = 0.0;
            if (r < n) {
                if (KP > 0) load_row<KP>(u.P + r * KP, p[t]);
                if (hx) load_row<K>(u.Xin + r * K, x[t]);
                if (u.W) load_row<K>(u.W + r * K, w[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < FU; ++t) {
            const int64_t r = r0 + t * S;
            if (r >= n) break;
            double o[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < KP; ++q) acc = fma(p[t][q], c[q][j], acc);
                double v = u.s * acc;
                if (hx) v = fma(u.a, x[t][j], v);
                if (u.W) v = fma(wv, w[t][j], v);
                o[j] = v;
            }
            double* op = u.out + r * K;
            if constexpr (K == 4) {
                reinterpret_cast<double2*>(op)[0] = make_double2(o[0], o[1]);
                reinterpret_cast<double2*>(op)[1] = make_double2(o[2], o[3]);
            } else if constexpr (K == 2) {
                reinterpret_cast<double2*>(op)[0] = make_double2(o[0], o[1]);
            } else {
#pragma unroll
                for (int j = 0; j < K; ++j) op[j] = o[j];
            }
        }
    }
}

// Gram k = 1, 2 (ka = kb = k): the operands are read as flat arrays of 32-byte vectors (4 / k
// rows per load), so every load instruction moves 32 bytes instead of 8 / 16 and one trip over
// c2 keeps the whole operand in flight (ncu c2, cold L2: k = 1 / 2 11.0 / 12.6 -> 10.1 / 11.8 us;
// the same for the update measured slower, 7.6 -> 9.2 us at k = 1, and is not used).  Rows beyond the last full vector (n k % 4 doubles: whole
// rows) are done by the first warp.  Same fixed-order reduction as gram_flat_kernel.
__device__ __forceinline__ void ld4(const double* __restrict__ p, double (&v)[4]) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

template <int K>
__global__ void __launch_bounds__(FT) gram_vec_kernel(int64_t n, const double* __restrict__ X,
                                                      const double* __restrict__ Y, double* __restrict__ G,
                                                      double* __restrict__ part, int* __restrict__ ticket) {
    constexpr int NO = K * K;
    double acc[K][K];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) acc[a][b] = 0.0;
    const int64_t nv = n * K / 4;   // full 32-byte vectors
    const int64_t S = (int64_t)gridDim.x * FT;
    for (int64_t v0 = (int64_t)blockIdx.x * FT + threadIdx.x; v0 < nv; v0 += FU * S) {
        double x[FU][4], y[FU][4];
#pragma unroll
        for (int u = 0; u < FU; ++u) {
            const int64_t v = v0 + u * S;
#pragma unroll
            for (int j = 0; j < 4; ++j) x[u][j] = y[u][j] = 0.0;
            if (v < nv) {
                ld4(X + 4 * v, x[u]);
                ld4(Y + 4 * v, y[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < FU; ++u)
#pragma unroll
            for (int r = 0; r < 4 / K; ++r)
#pragma unroll
                for (int a = 0; a < K; ++a)
#pragma unroll
                    for (int b = 0; b < K; ++b) acc[a][b] = fma(x[u][r * K + a], y[u][r * K + b], acc[a][b]);
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {   // ragged rows
        for (int64_t r = nv * 4 / K + threadIdx.x; r < n; r += 32)
#pragma unroll
            for (int a = 0; a < K; ++a)
#pragma unroll
                for (int b = 0; b < K; ++b) acc[a][b] = fma(X[r * K + a], Y[r * K + b], acc[a][b]);
    }
    __shared__ double s_w[FT / 32][NO];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
            double v = acc[a][b];
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
            if (lane == 0) s_w[warp][a * K + b] = v;
        }
    __syncthreads();
    if (threadIdx.x < NO) {
        double v = s_w[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < FT / 32; ++w) v += s_w[w][threadIdx.x];
        part[(int64_t)blockIdx.x * NO + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double f[NO];
#pragma unroll
    for (int q = 0; q < NO; ++q) f[q] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += FT)
#pragma unroll
        for (int q = 0; q < NO; ++q) f[q] += __ldcg(part + (int64_t)b * NO + q);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NO; ++q) {
        double v = f[q];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) s_w[warp][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < NO) {
        double v = s_w[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < FT / 32; ++w) v += s_w[w][threadIdx.x];
        G[threadIdx.x] = v;
    }
    if (threadIdx.x == 0) *ticket = 0;
}

// grid: at most 2 blocks of 512 per SM (4 rows per thread per trip keep >= 40 MB of loads in
// flight); few blocks keep the serial tail short -- one partial row per thread of the last block
int flat_grid(int64_t n, int num_sms) {
    const int64_t want = (n + (int64_t)FT * FU - 1) / ((int64_t)FT * FU);
    const int64_t cap = (int64_t)2 * num_sms;
    return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

size_t flat_part_doubles(int num_sms) { return (size_t)2 * num_sms * 16; }

bool launch_gram_flat(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                      double* G, double* part, int* ticket, int num_sms, cudaStream_t st) {
    if (n <= 0 || ka > 4 || kb > 4 || ldx != ka || ldy != kb) return false;
    if ((ka % 2 == 0 && ((uintptr_t)X & 15)) || (kb % 2 == 0 && ((uintptr_t)Y & 15))) return false;
    if ((ka == 4 && ((uintptr_t)X & 31)) || (kb == 4 && ((uintptr_t)Y & 31))) return false;
    if (ka == kb && ka <= 2 && !((uintptr_t)X & 31) && !((uintptr_t)Y & 31)) {   // 32-byte vectors
        const int grid = flat_grid(n * ka / 4, num_sms);
        if (ka == 1) BK_KERNEL(gram_vec_kernel<1><<<grid, FT, 0, st>>>(n, X, Y, G, part, ticket));
        else BK_KERNEL(gram_vec_kernel<2><<<grid, FT, 0, st>>>(n, X, Y, G, part, ticket));
        return true;
    }
    const int grid = flat_grid(n, num_sms);
#define BK_GF(A, B) \
    if (ka == A && kb == B) { BK_KERNEL(gram_flat_kernel<A, B><<<grid, FT, 0, st>>>(n, X, Y, G, part, ticket)); return true; }
    BK_GF(1, 1) BK_GF(1, 2) BK_GF(1, 3) BK_GF(1, 4) BK_GF(2, 1) BK_GF(2, 2) BK_GF(2, 3) BK_GF(2, 4)
    BK_GF(3, 1) BK_GF(3, 2) BK_GF(3, 3) BK_GF(3, 4) BK_GF(4, 1) BK_GF(4, 2) BK_GF(4, 3) BK_GF(4, 4)
#undef BK_GF
    return false;
}

bool launch_update_flat(const UpdArgs& u, int num_sms, cudaStream_t st) {
    if (u.n <= 0 || u.k > 4 || u.kp > 4 || u.kp < 0) return false;
    if (u.ldo != u.k || (u.kp > 0 && u.ldp != u.kp) || (u.a != 0.0 && u.Xin && u.ldxin != u.k) ||
        (u.W && u.ldw != u.k))
        return false;
    // (in place, out == P, is safe: each thread reads whole rows of P before writing them)
    if (u.kp > 0 && (const double*)u.out == u.P && u.ldo != u.kp) return false;
    if (u.kp == 0 && (u.a == 0.0 || !u.Xin) && !u.W) return false;
    auto al = [](const void* p, int w) {
        return !p || (w == 4 ? ((uintptr_t)p & 31) == 0 : (w == 2 ? ((uintptr_t)p & 15) == 0 : true));
    };
    if (!al(u.out, u.k) || !al(u.kp > 0 ? u.P : nullptr, u.kp) || !al(u.a != 0.0 ? u.Xin : nullptr, u.k) ||
        !al(u.W, u.k))
        return false;
    if (u.out && u.k == 4 && ((uintptr_t)u.out & 15)) return false;
    const int grid = flat_grid(u.n, num_sms);
#define BK_UF(K, KP) \
    if (u.k == K && u.kp == KP) { BK_KERNEL(upd_flat_kernel<K, KP><<<grid, FT, 0, st>>>(u)); return true; }
    BK_UF(1, 0) BK_UF(1, 1) BK_UF(1, 2) BK_UF(1, 3) BK_UF(1, 4)
    BK_UF(2, 0) BK_UF(2, 1) BK_UF(2, 2) BK_UF(2, 3) BK_UF(2, 4)
    BK_UF(3, 0) BK_UF(3, 1) BK_UF(3, 2) BK_UF(3, 3) BK_UF(3, 4)
    BK_UF(4, 0) BK_UF(4, 1) BK_UF(4, 2) BK_UF(4, 3) BK_UF(4, 4)
#undef BK_UF
    return false;
}

}  // namespace bk
