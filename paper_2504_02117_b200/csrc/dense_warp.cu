// dense_warp.cu -- a4 small dense k x k stage as single-warp kernels (k <= 32).
//
// One warp, matrices in shared memory (padded rows, conflict-free), lanes work
// on rows (elimination) or on right-hand-side columns (substitution), loops
// rolled (compact code: a fully unrolled register version was 57 K SASS
// instructions and I-cache bound), only __syncwarp between steps (the
// 256-thread CTA versions in dense.cu spend ~100 block barriers per call).
// Breakdown is a status (DevStatus), never a crash (R6).
#include "bk_internal.h"
#include "dense_dev.cuh"

namespace bk {
namespace {

using dd::KM;
using dd::LD;
using dd::wmax;

// LU with partial pivoting (explicit row swaps), Out = G^{-1} (sign Rhs)
// (dense_dev.cuh lu_solve_warp); LUo / pivo keep the factors for lu_resolve_w.
__global__ void __launch_bounds__(32) lu_solve_w(int defer, const double* __restrict__ G, const double* __restrict__ Rhs,
                                                 double* __restrict__ Out, int k, int nrhs, double sign, double tol,
                                                 DevStatus* st, double* __restrict__ LUo, int* __restrict__ pivo) {
    __shared__ double A[KM * LD], B[KM * LD];
    __shared__ int s_piv[KM];
    dd::lu_solve_warp(defer, G, Rhs, Out, k, nrhs, sign, tol, st, LUo, pivo, A, B, s_piv);
}

// Out = G^{-1} (sign Rhs) from lu_solve_w's factors (getrs).
__global__ void __launch_bounds__(32) lu_resolve_w(const double* __restrict__ LU, const int* __restrict__ piv,
                                                   const double* __restrict__ Rhs, double* __restrict__ Out, int k,
                                                   int nrhs, double sign, DevStatus* st) {
    __shared__ double A[KM * LD], B[KM * LD];
    dd::lu_resolve_warp(LU, piv, Rhs, Out, k, nrhs, sign, st, A, B);
}

// Cholesky of A (lower part, lane = row); returns breakdown column or -1.
__device__ int chol_w(double* A, int k, double tol) {
    const int l = threadIdx.x;
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

// Out = G^{-1} Rhs by Cholesky: L w = Rhs, L^T z = w (lane = rhs column).
__global__ void __launch_bounds__(32) chol_solve_w(const double* __restrict__ G, const double* __restrict__ Rhs,
                                                   double* __restrict__ Out, int k, int nrhs, double tol,
                                                   DevStatus* st) {
    __shared__ double A[KM * LD], B[KM * LD];
    if (st && st->halt) return;
    const int l = threadIdx.x;
    for (int r = 0; r < k; ++r) {
        if (l < k) A[r * LD + l] = G[r * k + l];
        if (l < nrhs) B[r * LD + l] = Rhs[r * nrhs + l];
    }
    __syncwarp();
    const int fail = chol_w(A, k, tol);
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

// CholQR factor: G = R^T R (R = L^T), Rinv = R^{-1} (lane = column), Rprod = R Rprev.
__global__ void __launch_bounds__(32) chol_qr_w(const double* __restrict__ G, double* __restrict__ R,
                                                double* __restrict__ Rinv, const double* __restrict__ Rprev,
                                                double* __restrict__ Rprod, int k, double tol, DevStatus* st) {
    __shared__ double A[KM * LD], Z[KM * LD];
    if (st && st->halt) return;
    const int l = threadIdx.x;
    for (int r = 0; r < k; ++r)
        if (l < k) A[r * LD + l] = G[r * k + l];
    __syncwarp();
    const int fail = chol_w(A, k, tol);
    if (fail >= 0) {
        if (l == 0 && st) { st->breakdown_col = fail; st->halt = 1; }
        return;
    }
    if (l < k) {
        // R[r][c] = L[c][r] (c >= r); column l of R^{-1}: R z = e_l, R[q][p] = L[p][q]
#pragma unroll 1
        for (int q = k - 1; q >= 0; --q) {
            double v = (q == l) ? 1.0 : 0.0;
#pragma unroll 4
            for (int p = q + 1; p < k; ++p) v = fma(-A[p * LD + q], Z[p * LD + l], v);
            Z[q * LD + l] = v / A[q * LD + q];
        }
        for (int q = 0; q < k; ++q) {
            Rinv[q * k + l] = (q <= l) ? Z[q * LD + l] : 0.0;
            if (R) R[q * k + l] = (l >= q) ? A[l * LD + q] : 0.0;
        }
        if (Rprev && Rprod) {
            for (int r = 0; r < k; ++r) {
                double v = 0.0;
                for (int q = r; q < k; ++q) v = fma(A[q * LD + r], Rprev[q * k + l], v);
                Rprod[r * k + l] = v;
            }
        }
    }
}

// a fused pass's k x k epilogue run on its own (dense_dev.cuh run_small_epi)
__global__ void __launch_bounds__(32) small_epi_w(const SmallEpi e) {
    __shared__ double scr[dd::SCRATCH_DOUBLES];
    dd::run_small_epi(e, scr);
}

}  // namespace

void sd_small_epi(const SmallEpi& e, cudaStream_t s) { BK_KERNEL(small_epi_w<<<1, 32, 0, s>>>(e)); }

void sdw_lu_solve(const double* G, const double* Rhs, double* Out, int k, int nrhs, double sign, double tol,
                  DevStatus* st, cudaStream_t s, int defer, double* LUo, int* pivo) {
    BK_KERNEL(lu_solve_w<<<1, 32, 0, s>>>(defer, G, Rhs, Out, k, nrhs, sign, tol, st, LUo, pivo));
}

void sd_lu_resolve(const double* LU, const int* piv, const double* Rhs, double* Out, int k, int nrhs, double sign,
                   DevStatus* st, cudaStream_t s) {
    BK_KERNEL(lu_resolve_w<<<1, 32, 0, s>>>(LU, piv, Rhs, Out, k, nrhs, sign, st));
}

void sdw_chol_solve(const double* G, const double* Rhs, double* Out, int k, int nrhs, double tol, DevStatus* st,
                    cudaStream_t s) {
    BK_KERNEL(chol_solve_w<<<1, 32, 0, s>>>(G, Rhs, Out, k, nrhs, tol, st));
}

void sdw_chol_qr(const double* G, double* R, double* Rinv, const double* Rprev, double* Rprod, int k, double tol,
                 DevStatus* st, cudaStream_t s) {
    BK_KERNEL(chol_qr_w<<<1, 32, 0, s>>>(G, R, Rinv, Rprev, Rprod, k, tol, st));
}

}  // namespace bk
