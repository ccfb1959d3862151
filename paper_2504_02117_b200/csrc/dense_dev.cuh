// dense_dev.cuh -- single-warp device routines of the a4 small dense k x k stage
// (k <= 32), shared by the one-warp kernels (dense_warp.cu) and the epilogues of
// the fused reduction kernels (stream.cu: the last CTA of a Gram pass solves
// with the k x k result it just produced).  Internal header; nothing here is
// shared with oracle/.  Breakdown is a status (DevStatus), never a crash
// (R6).
#pragma once

#include "bk_internal.h"

namespace bk {
namespace dd {

constexpr int KM = BK_MAX_K;
constexpr int LD = KM + 1;
constexpr int SCRATCH_DOUBLES = 3 * KM * LD + KM;   // A, B, pivots, T (kind 6)

__device__ __forceinline__ double wmax(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, m));
    return v;
}

// LU with partial pivoting (explicit row swaps), Out = G^{-1} (sign Rhs).
// rows < k of a k x ncols row-major matrix (scaled) into smem, all loads in flight first
__device__ __forceinline__ void load_rows_w(const double* __restrict__ src, double* dst, int k, int ncols, double scale) {
    const int l = threadIdx.x & 31;
    double v[KM];
#pragma unroll
    for (int r = 0; r < KM; ++r) v[r] = (r < k && l < ncols) ? src[r * ncols + l] : 0.0;
#pragma unroll
    for (int r = 0; r < KM; ++r)
        if (r < k && l < ncols) dst[r * LD + l] = scale * v[r];
}

// LU with partial pivoting (explicit row swaps), Out = G^{-1} (sign Rhs).
// LUo / pivo (optional): the factors (P G = L U, unit L below the diagonal,
// getrf layout) and the pivot row of each step, for lu_resolve_w.
// Column-parallel elimination: lane c owns column c of [A | B] (k + nrhs <= 64: two
// columns per lane), so step j costs k - j - 1 fused updates per lane; pivots and
// 1/U_jj are broadcast.
__device__ __forceinline__ void lu_solve_warp(int defer, const double* __restrict__ G, const double* __restrict__ Rhs,
                                              double* __restrict__ Out, int k, int nrhs, double sign, double tol,
                                              DevStatus* st, double* __restrict__ LUo, int* __restrict__ pivo,
                                              double* A, double* B, int* s_piv) {
    if (st && st->halt) return;
    const int l = threadIdx.x & 31;
    load_rows_w(G, A, k, k, 1.0);
    load_rows_w(Rhs, B, k, nrhs, sign);
    __syncwarp();
    double mx = 0.0;
    for (int r = 0; r < k; ++r)
        if (l < k) mx = fmax(mx, fabs(A[r * LD + l]));
    mx = wmax(mx);
    if (!(mx > 0.0)) mx = 2.2250738585072014e-308;
    // the two columns of lane l: A column l (if l < k) and B column l (if l < nrhs)
    const bool ha = l < k, hb = l < nrhs;
#pragma unroll 1
    for (int j = 0; j < k; ++j) {
        double v = (l >= j && l < k) ? fabs(A[l * LD + j]) : -1.0;
        int p = l;
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, m);
            const int op = __shfl_xor_sync(0xffffffffu, p, m);
            if (ov > v || (ov == v && op < p)) { v = ov; p = op; }
        }
        if (!(v > tol * mx)) {
            if (l == 0 && st) {
                if (defer) st->pending_bd = j + 1;
                else { st->breakdown_col = j; st->halt = 1; }
            }
            return;
        }
        if (l == 0) s_piv[j] = p;
        if (p != j) {   // lane l swaps its columns' entries of rows j and p
            if (ha) { const double t = A[j * LD + l]; A[j * LD + l] = A[p * LD + l]; A[p * LD + l] = t; }
            if (hb) { const double t = B[j * LD + l]; B[j * LD + l] = B[p * LD + l]; B[p * LD + l] = t; }
        }
        __syncwarp();
        const double inv = 1.0 / A[j * LD + j];
        const double aj = (ha && l > j) ? A[j * LD + l] : 0.0, bj = hb ? B[j * LD + l] : 0.0;
#pragma unroll 4
        for (int r = j + 1; r < k; ++r) {
            const double f = A[r * LD + j] * inv;   // multiplier of row r (broadcast)
            if (ha && l > j) A[r * LD + l] = fma(-f, aj, A[r * LD + l]);
            if (hb) B[r * LD + l] = fma(-f, bj, B[r * LD + l]);
        }
        __syncwarp();
        if (l > j && l < k) A[l * LD + j] *= inv;   // L multiplier (getrf layout), lane = row
        __syncwarp();
    }
    // back substitution, lane = right-hand-side column (solution overwrites B); the 1/U_ii are
    // formed in parallel (lane i) and broadcast, two partial sums halve the dependent chain
    const double dinv = l < k ? 1.0 / A[l * LD + l] : 0.0;
#pragma unroll 1
    for (int i = k - 1; i >= 0; --i) {
        const double di = __shfl_sync(0xffffffffu, dinv, i);
        if (l < nrhs) {
            double v0 = B[i * LD + l], v1 = 0.0;
            int q = i + 1;
            for (; q + 1 < k; q += 2) {
                v0 = fma(-A[i * LD + q], B[q * LD + l], v0);
                v1 = fma(-A[i * LD + q + 1], B[(q + 1) * LD + l], v1);
            }
            if (q < k) v0 = fma(-A[i * LD + q], B[q * LD + l], v0);
            B[i * LD + l] = (v0 + v1) * di;
        }
    }
    if (l < nrhs)
        for (int i = 0; i < k; ++i) Out[i * nrhs + l] = B[i * LD + l];
    if (LUo && l < k)
        for (int r = 0; r < k; ++r) LUo[r * k + l] = A[r * LD + l];
    if (pivo && l < k) pivo[l] = s_piv[l];
}

// Out = G^{-1} (sign Rhs) from lu_solve_w's factors (getrs): b <- P b, L y = b, U x = y.
__device__ __forceinline__ void lu_resolve_warp(const double* __restrict__ LU, const int* __restrict__ piv,
                                                const double* __restrict__ Rhs, double* __restrict__ Out, int k,
                                                int nrhs, double sign, DevStatus* st, double* A, double* B) {
    if (st && st->halt) return;
    const int l = threadIdx.x & 31;
    load_rows_w(LU, A, k, k, 1.0);
    load_rows_w(Rhs, B, k, nrhs, sign);
    __syncwarp();
    if (l < nrhs) {
#pragma unroll 1
        for (int j = 0; j < k; ++j) {   // b <- P b (all interchanges, in order: getrs)
            const int p = piv[j];
            if (p != j) { const double t = B[j * LD + l]; B[j * LD + l] = B[p * LD + l]; B[p * LD + l] = t; }
        }
#pragma unroll 1
        for (int j = 0; j < k; ++j) {   // L y = b (unit lower, final row order)
            const double bj = B[j * LD + l];
            for (int i = j + 1; i < k; ++i) B[i * LD + l] = fma(-A[i * LD + j], bj, B[i * LD + l]);
        }
    }
    const double dinv = l < k ? 1.0 / A[l * LD + l] : 0.0;   // 1/U_ii, broadcast below
#pragma unroll 1
    for (int i = k - 1; i >= 0; --i) {
        const double di = __shfl_sync(0xffffffffu, dinv, i);
        if (l < nrhs) {
            double v0 = B[i * LD + l], v1 = 0.0;
            int q = i + 1;
            for (; q + 1 < k; q += 2) {
                v0 = fma(-A[i * LD + q], B[q * LD + l], v0);
                v1 = fma(-A[i * LD + q + 1], B[(q + 1) * LD + l], v1);
            }
            if (q < k) v0 = fma(-A[i * LD + q], B[q * LD + l], v0);
            B[i * LD + l] = (v0 + v1) * di;
        }
    }
    if (l < nrhs)
        for (int i = 0; i < k; ++i) Out[i * nrhs + l] = B[i * LD + l];
}

// Cholesky of A (lower part, lane = row) in place; returns the breakdown column or -1.
__device__ __forceinline__ int chol_warp(double* A, int k, double tol) {
    const int l = threadIdx.x & 31;
    double scale = wmax(l < k ? fabs(A[l * LD + l]) : 0.0);
    if (!(scale > 0.0)) scale = 2.2250738585072014e-308;
#pragma unroll 1
    for (int j = 0; j < k; ++j) {
        const double d = A[j * LD + j];
        if (!(d > tol * scale)) return j;
        const double ljj = sqrt(d);
        __syncwarp();
        if (l == j) A[j * LD + j] = ljj;
        if (l > j && l < k) A[l * LD + j] /= ljj;
        __syncwarp();
        if (l > j && l < k) {
            const double lij = A[l * LD + j];
#pragma unroll 4
            for (int c = j + 1; c <= l; ++c) A[l * LD + c] = fma(-lij, A[c * LD + j], A[l * LD + c]);
        }
        __syncwarp();
    }
    return -1;
}

// Out = G^{-1} Rhs by Cholesky (G SPD k x k, Rhs k x nrhs); breakdown -> status
__device__ __forceinline__ void chol_solve_warp(const double* __restrict__ G, const double* __restrict__ Rhs,
                                                double* __restrict__ Out, int k, int nrhs, double tol,
                                                DevStatus* st, double* A, double* B) {
    if (st && st->halt) return;
    const int l = threadIdx.x & 31;
    load_rows_w(G, A, k, k, 1.0);
    load_rows_w(Rhs, B, k, nrhs, 1.0);
    __syncwarp();
    const int fail = chol_warp(A, k, tol);
    if (fail >= 0) {
        if (l == 0 && st) { st->breakdown_col = fail; st->halt = 1; }
        return;
    }
    if (l < nrhs) {
#pragma unroll 1
        for (int i = 0; i < k; ++i) {
            double v = B[i * LD + l];
#pragma unroll 4
            for (int q = 0; q < i; ++q) v = fma(-A[i * LD + q], B[q * LD + l], v);
            B[i * LD + l] = v / A[i * LD + i];
        }
#pragma unroll 1
        for (int i = k - 1; i >= 0; --i) {
            double v = B[i * LD + l];
#pragma unroll 4
            for (int q = i + 1; q < k; ++q) v = fma(-A[q * LD + i], B[q * LD + l], v);
            B[i * LD + l] = v / A[i * LD + i];
        }
        for (int i = 0; i < k; ++i) Out[i * nrhs + l] = B[i * LD + l];
    }
}

// BiCGStab omega = sum ts / sum tt (lane 0); tt <= 0 is a breakdown
__device__ __forceinline__ void omega_dev(const double* ts, const double* tt, int k, int stride, DevStatus* st) {
    if ((threadIdx.x & 31) != 0 || st->halt) return;
    double a = 0.0, b = 0.0;
    for (int c = 0; c < k; ++c) { a += ts[c * stride]; b += tt[c * stride]; }
    if (!(b > 0.0)) { st->breakdown_col = 0; st->halt = 1; return; }
    st->omega = a / b;
    st->neg_omega = -(a / b);
}

// convergence test (lane 0): rel_c = sqrt(max(g_c, 0)) / r0_c; init stores r0
__device__ __forceinline__ void conv_check_dev(const double* g, int gstride, int k, double rtol, int conv_mode,
                                               int init, DevStatus* st) {
    if ((threadIdx.x & 31) != 0) return;
    if (init) {
        for (int c = 0; c < k; ++c) st->r0[c] = sqrt(fmax(g[c * gstride], 0.0));
        return;
    }
    if (st->halt) return;
    bool ok = true;
    for (int c = 0; c < k; ++c) {
        const double r0 = st->r0[c];
        const double rel = sqrt(fmax(g[c * gstride], 0.0)) / (r0 > 0.0 ? r0 : 1.0);
        st->relres[c] = rel;
        if (conv_mode == BK_CONV_FIRST ? (c == 0 && !(rel <= rtol)) : !(rel <= rtol)) ok = false;
    }
    st->iter += 1;
    if (ok) { st->converged = 1; st->halt = 1; }
    else if (st->pending_bd) { st->breakdown_col = st->pending_bd - 1; st->halt = 1; }
}

// Epilogue of a fused reduction pass (warp 0 of the CTA that wrote the final
// k x k results; the caller has made those writes visible with a CTA barrier).
__device__ __forceinline__ void run_small_epi(const SmallEpi& e, double* scratch) {
    if (e.kind == 0) return;
    double* A = scratch;
    double* B = A + KM * LD;
    int* piv = reinterpret_cast<int*>(B + KM * LD);
    if (e.kind == 1) {
        lu_solve_warp(0, e.G, e.Rhs, e.Out, e.k, e.k, e.sign, e.tol, e.st, e.LU, e.piv, A, B, piv);
    } else if (e.kind == 2) {
        omega_dev(e.ts, e.tt, e.k, 1, e.st);
        __syncwarp();
        lu_resolve_warp(e.LU, e.piv, e.Rhs, e.Out, e.k, e.k, e.sign, e.st, A, B);
    } else if (e.kind == 3) {
        conv_check_dev(e.g, 1, e.k, e.rtol, e.conv_mode, 0, e.st);
    } else if (e.kind == 4) {   // block CG alpha: Out = G^{-1} Rhs (Cholesky)
        chol_solve_warp(e.G, e.Rhs, e.Out, e.k, e.k, e.tol, e.st, A, B);
    } else if (e.kind == 5) {   // block CG: test on diag(g = R^T R new), beta = Rhs^{-1} g, Rhs <- g
        conv_check_dev(e.g, e.k + 1, e.k, e.rtol, e.conv_mode, 0, e.st);
        __syncwarp();
        chol_solve_warp(e.Rhs, e.g, e.Out, e.k, e.k, e.tol, e.st, A, B);
        __syncwarp();
        double* rz = const_cast<double*>(e.Rhs);   // roll R^T R for the next iteration
        for (int t = threadIdx.x & 31; t < e.k * e.k; t += 32) rz[t] = e.g[t];
    } else if (e.kind == 6 || e.kind == 7) {
        // single-reduction block CG (oracle O11) from the one reduction pass over [R, W = A R]:
        // g = R^T R (new), G = R^T W, Rhs = R^T R of the previous iteration (rolled here),
        // S = the S state (P^T A P), Out = alpha, Out2 = beta.
        //   7 (setup): r0 from diag(g); S = G; alpha = S^{-1} g; beta = 0
        //   6: test on diag(g); beta = Rhs^{-1} g; S = G - beta^T S beta; alpha = S^{-1} g
        const int l = threadIdx.x & 31, k = e.k;
        conv_check_dev(e.g, k + 1, k, e.rtol, e.conv_mode, e.kind == 7, e.st);
        __syncwarp();
        if (e.st->halt) return;
        if (e.kind == 7) {
            for (int t = l; t < k * k; t += 32) { e.S[t] = e.G[t]; e.Out2[t] = 0.0; }
        } else {
            chol_solve_warp(e.Rhs, e.g, e.Out2, k, k, e.tol, e.st, A, B);   // B = beta (k x k, LD)
            __syncwarp();
            if (e.st->halt) return;
            double* T = B + KM * LD + KM;
            load_rows_w(e.S, A, k, k, 1.0);
            __syncwarp();
            if (l < k) {   // T = S beta, lane = column
                for (int r = 0; r < k; ++r) {
                    double v = 0.0;
                    for (int q = 0; q < k; ++q) v = fma(A[r * LD + q], B[q * LD + l], v);
                    T[r * LD + l] = v;
                }
            }
            __syncwarp();
            if (l < k) {   // S = G - beta^T T
                for (int r = 0; r < k; ++r) {
                    double v = 0.0;
                    for (int q = 0; q < k; ++q) v = fma(B[q * LD + r], T[q * LD + l], v);
                    e.S[r * k + l] = e.G[r * k + l] - v;
                }
            }
        }
        __syncwarp();
        chol_solve_warp(e.S, e.g, e.Out, k, k, e.tol, e.st, A, B);
        __syncwarp();
        double* rz = const_cast<double*>(e.Rhs);
        for (int t = l; t < k * k; t += 32) rz[t] = e.g[t];
    }
}

}  // namespace dd
}  // namespace bk
