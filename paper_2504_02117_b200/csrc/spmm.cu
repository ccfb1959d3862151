// spmm.cu -- a1: block operator apply  Y = alpha (A X) C + beta Y  on sm_100a.
//
// PAPER.md §3: the BOP kernel "Y <- A X" loads the matrix once for
// all k columns.  B200 mapping:
//  * one CTA = one tile of TR consecutive rows; the tile's row pointers,
//    column ids and values (a contiguous CSR range) are streamed from HBM
//    exactly once with coalesced 16-byte loads into shared memory;
//  * a group of LANES = KP/VEC threads owns one row; lane l holds columns
//    [l*VEC, l*VEC+VEC) (VEC = 2 -> 16-byte vector gathers of X);
//  * X rows are gathered through L1/L2 (neighbouring rows of a stencil hit the
//    same lines), Y is written once with streaming (evict-first) stores;
//  * the optional k x k_out coupling C is applied in the epilogue
//    from shared memory, so the coupled apply costs no extra HBM pass.
#include "bk_internal.h"

namespace bk {
namespace {

constexpr int kThreads = 256;
constexpr int kTileRows = 256;   // rows per CTA tile
constexpr int kCap = 2048;       // staged nonzeros per tile (fallback: direct loads)

__device__ __forceinline__ void ld_x(const double* p, double (&x)[1]) { x[0] = __ldg(p); }
__device__ __forceinline__ void ld_x(const double* p, double (&x)[2]) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    x[0] = v.x; x[1] = v.y;
}
__device__ __forceinline__ void ld_x4(const double* p, double (&x)[4]) {
    double2 v0 = __ldg(reinterpret_cast<const double2*>(p));
    double2 v1 = __ldg(reinterpret_cast<const double2*>(p + 2));
    x[0] = v0.x; x[1] = v0.y; x[2] = v1.x; x[3] = v1.y;
}
__device__ __forceinline__ void ld_x(const double* p, double (&x)[4]) { ld_x4(p, x); }

// streaming 16-byte load of CSR data (read once: do not pollute L1)
__device__ __forceinline__ int4 ld_stream_i4(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

template <int VEC>
__device__ __forceinline__ void st_y(double* p, const double (&v)[VEC], int valid) {
    if (VEC == 2 && valid == 2) {
        __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
    } else {
#pragma unroll
        for (int t = 0; t < VEC; ++t)
            if (t < valid) __stcs(p + t, v[t]);
    }
}

template <int KP, int VEC, bool HAS_C, bool GHOST>
__global__ void __launch_bounds__(kThreads)
bspmm_tile_kernel(const SpmmArgs a) {
    constexpr int LANES = KP / VEC;
    constexpr int RPP = kThreads / LANES;       // rows per pass
    constexpr int PASSES = kTileRows / RPP;
    __shared__ int32_t s_rp[kTileRows + 1];
    __shared__ __align__(16) int32_t s_col[kCap + 4];
    __shared__ __align__(16) double s_val[kCap + 4];
    __shared__ double s_C[HAS_C ? KP * KP : 1];
    __shared__ double s_t[HAS_C ? RPP * (KP + 1) : 1];

    const int tid = threadIdx.x;
    const int grp = tid / LANES;
    const int lane = tid % LANES;
    const int c0 = lane * VEC;
    const int k = a.k;
    const int kout = a.kout;

    if (HAS_C) {
        for (int i = tid; i < KP * KP; i += kThreads) {
            int r = i / KP, c = i % KP;
            s_C[i] = (r < k && c < kout) ? a.C[r * kout + c] : 0.0;
        }
    }
    const int64_t tile0 = a.row0 + (int64_t)blockIdx.x * kTileRows;
    const int nr = (int)((a.row0 + a.nrows - tile0) < kTileRows ? (a.row0 + a.nrows - tile0) : kTileRows);
    for (int i = tid; i <= nr; i += kThreads) s_rp[i] = a.rp[tile0 + i];
    __syncthreads();
    const int p0 = s_rp[0];
    const int nnz = s_rp[nr] - p0;
    const bool staged = nnz <= kCap;
    // aligned start so that the 16-byte vector loads are legal (arrays are
    // 256-byte aligned and padded by the library, see abi.cpp)
    const int pa = p0 & ~3;
    const int off = p0 - pa;
    if (staged) {
        const int n4 = (off + nnz + 3) >> 2;           // int4 / 2x double2 chunks
        const int4* gc = reinterpret_cast<const int4*>(a.col + pa);
        const double2* gv = reinterpret_cast<const double2*>(a.val + pa);
        int4* sc = reinterpret_cast<int4*>(s_col);
        double2* sv = reinterpret_cast<double2*>(s_val);
        for (int i = tid; i < n4; i += kThreads) {
            sc[i] = ld_stream_i4(gc + i);
            sv[2 * i] = ld_stream_d2(gv + 2 * i);
            sv[2 * i + 1] = ld_stream_d2(gv + 2 * i + 1);
        }
    }
    __syncthreads();

    const bool lane_in = c0 < k;
    for (int pass = 0; pass < PASSES; ++pass) {
        const int r = pass * RPP + grp;
        const bool active = r < nr;
        double acc[VEC];
#pragma unroll
        for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
        if (active) {
            const int s = s_rp[r] - p0, e = s_rp[r + 1] - p0;
            if (staged) {
                const int* scol = s_col + off;
                const double* sval = s_val + off;
                int p = s;
                for (; p + 1 < e; p += 2) {
                    const int ca = scol[p], cb = scol[p + 1];
                    const double va = sval[p], vb = sval[p + 1];
                    const double* xa = (GHOST && ca >= a.ncol_local)
                                           ? a.Xg + (int64_t)(ca - a.ncol_local) * a.ldg
                                           : a.X + (int64_t)ca * a.ldx;
                    const double* xb = (GHOST && cb >= a.ncol_local)
                                           ? a.Xg + (int64_t)(cb - a.ncol_local) * a.ldg
                                           : a.X + (int64_t)cb * a.ldx;
                    if (lane_in) {
                        double x0[VEC], x1[VEC];
                        ld_x(xa + c0, x0);
                        ld_x(xb + c0, x1);
#pragma unroll
                        for (int t = 0; t < VEC; ++t) acc[t] = fma(va, x0[t], acc[t]);
#pragma unroll
                        for (int t = 0; t < VEC; ++t) acc[t] = fma(vb, x1[t], acc[t]);
                    }
                }
                if (p < e) {
                    const int ca = scol[p];
                    const double va = sval[p];
                    const double* xa = (GHOST && ca >= a.ncol_local)
                                           ? a.Xg + (int64_t)(ca - a.ncol_local) * a.ldg
                                           : a.X + (int64_t)ca * a.ldx;
                    if (lane_in) {
                        double x0[VEC];
                        ld_x(xa + c0, x0);
#pragma unroll
                        for (int t = 0; t < VEC; ++t) acc[t] = fma(va, x0[t], acc[t]);
                    }
                }
            } else {
                for (int p = s; p < e; ++p) {
                    const int ca = __ldg(a.col + p0 + p);
                    const double va = __ldg(a.val + p0 + p);
                    const double* xa = (GHOST && ca >= a.ncol_local)
                                           ? a.Xg + (int64_t)(ca - a.ncol_local) * a.ldg
                                           : a.X + (int64_t)ca * a.ldx;
                    if (lane_in) {
                        double x0[VEC];
                        ld_x(xa + c0, x0);
#pragma unroll
                        for (int t = 0; t < VEC; ++t) acc[t] = fma(va, x0[t], acc[t]);
                    }
                }
            }
        }
        double out[VEC];
        if (HAS_C) {
            double* t_row = s_t + grp * (KP + 1);
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
            double* yp = a.Y + (tile0 + r) * a.ldy + c0;
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
}

// Explicit row list (boundary rows of a partitioned matrix): no staging.
template <int KP, int VEC, bool HAS_C, bool GHOST>
__global__ void __launch_bounds__(kThreads)
bspmm_rows_kernel(const SpmmArgs a) {
    constexpr int LANES = KP / VEC;
    constexpr int RPP = kThreads / LANES;
    __shared__ double s_C[HAS_C ? KP * KP : 1];
    __shared__ double s_t[HAS_C ? RPP * (KP + 1) : 1];
    const int tid = threadIdx.x, grp = tid / LANES, lane = tid % LANES, c0 = lane * VEC;
    const int k = a.k, kout = a.kout;
    if (HAS_C) {
        for (int i = tid; i < KP * KP; i += kThreads) {
            int r = i / KP, c = i % KP;
            s_C[i] = (r < k && c < kout) ? a.C[r * kout + c] : 0.0;
        }
        __syncthreads();
    }
    const int64_t idx = (int64_t)blockIdx.x * RPP + grp;
    const bool active = idx < a.nrows;
    const int64_t row = active ? (a.rows ? (int64_t)a.rows[idx] : a.row0 + idx) : 0;
    double acc[VEC];
#pragma unroll
    for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
    if (active && c0 < k) {
        for (int p = a.rp[row]; p < a.rp[row + 1]; ++p) {
            const int ca = __ldg(a.col + p);
            const double va = __ldg(a.val + p);
            const double* xa = (GHOST && ca >= a.ncol_local) ? a.Xg + (int64_t)(ca - a.ncol_local) * a.ldg
                                                             : a.X + (int64_t)ca * a.ldx;
            double x0[VEC];
            ld_x(xa + c0, x0);
#pragma unroll
            for (int t = 0; t < VEC; ++t) acc[t] = fma(va, x0[t], acc[t]);
        }
    }
    double out[VEC];
    if (HAS_C) {
        double* t_row = s_t + grp * (KP + 1);
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
    } else {
#pragma unroll
        for (int t = 0; t < VEC; ++t) out[t] = acc[t];
    }
    if (active && c0 < kout) {
        double* yp = a.Y + row * a.ldy + c0;
        const int valid = min(VEC, kout - c0);
        double v[VEC];
#pragma unroll
        for (int t = 0; t < VEC; ++t)
            v[t] = (t < valid) ? (a.beta != 0.0 ? a.alpha * out[t] + a.beta * yp[t] : a.alpha * out[t]) : 0.0;
        st_y<VEC>(yp, v, valid);
    }
}

template <int KP, int VEC, bool HAS_C, bool GHOST>
void launch_t(const SpmmArgs& a, cudaStream_t st) {
    if (a.nrows <= 0) return;
    if (a.rows) {
        constexpr int RPP = kThreads / (KP / VEC);
        unsigned grid = (unsigned)((a.nrows + RPP - 1) / RPP);
        BK_KERNEL(bspmm_rows_kernel<KP, VEC, HAS_C, GHOST><<<grid, kThreads, 0, st>>>(a));
    } else {
        unsigned grid = (unsigned)((a.nrows + kTileRows - 1) / kTileRows);
        BK_KERNEL(bspmm_tile_kernel<KP, VEC, HAS_C, GHOST><<<grid, kThreads, 0, st>>>(a));
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

template <int KP>
void launch_k(const SpmmArgs& a, cudaStream_t st, bool vec2) {
    if constexpr (KP >= 2) {
        if (vec2) return launch_kv<KP, 2>(a, st);
    }
    launch_kv<KP, 1>(a, st);
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

}  // namespace bk
