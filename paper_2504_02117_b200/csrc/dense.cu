// dense.cu -- a4: the small dense k x k stage of the block Krylov iteration.
//
// Cholesky / LU solves of the k x k block coefficient systems, CholQR factors,
// the convergence test and the block-GMRES least-squares update.  O(k^3)
// flops (k <= 32), negligible work but on the critical path of every
// iteration, so each runs as ONE CTA on the device, redundantly on every rank
// (inputs are bitwise identical after the Gram allreduce), and never goes
// through the host.  Breakdown is reported through DevStatus (status, not a
// crash: SPEC S:129; reading R6).
#include "bk_internal.h"

namespace bk {
namespace {

constexpr int KM = BK_MAX_K;       // 32
constexpr int LD = KM + 1;         // padded smem leading dim

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

// Right-looking Cholesky of s (k x k, lower part used): s = L L^T in place
// (lower).  Returns breakdown column or -1.  All threads of the CTA call it.
__device__ int chol_lower_inplace(double* s, int k, double tol) {
    __shared__ int s_fail;
    __shared__ double s_scale;
    const int tid = threadIdx.x, nt = blockDim.x;
    if (tid == 0) {
        double m = 0.0;
        for (int i = 0; i < k; ++i) m = fmax(m, fabs(s[i * LD + i]));
        s_scale = m > 0.0 ? m : 2.2250738585072014e-308;
        s_fail = -1;
    }
    __syncthreads();
    for (int j = 0; j < k; ++j) {
        if (tid == 0) {
            const double d = s[j * LD + j];
            if (!(d > tol * s_scale)) s_fail = j;
            else s[j * LD + j] = sqrt(d);
        }
        __syncthreads();
        if (s_fail >= 0) return s_fail;
        const double piv = s[j * LD + j];
        for (int i = j + 1 + tid; i < k; i += nt) s[i * LD + j] /= piv;
        __syncthreads();
        // trailing update of the lower triangle: s[i][c] -= L[i][j] L[c][j], j < c <= i
        const int m = k - j - 1;
        for (int t = tid; t < m * m; t += nt) {
            const int i = j + 1 + t / m, c = j + 1 + t % m;
            if (c <= i) s[i * LD + c] = fma(-s[i * LD + j], s[c * LD + j], s[i * LD + c]);
        }
        __syncthreads();
    }
    return -1;
}

__global__ void chol_solve_kernel(const double* __restrict__ G, const double* __restrict__ Rhs,
                                  double* __restrict__ Out, int k, int nrhs, double tol, DevStatus* st) {
    __shared__ double s[KM * LD];
    __shared__ double b[KM * LD];
    if (st && st->halt) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < k * k; t += nt) s[(t / k) * LD + t % k] = G[t];
    for (int t = tid; t < k * nrhs; t += nt) b[(t / nrhs) * LD + t % nrhs] = Rhs[t];
    __syncthreads();
    const int fail = chol_lower_inplace(s, k, tol);
    if (fail >= 0) {
        if (tid == 0 && st) { st->breakdown_col = fail; st->halt = 1; }
        return;
    }
    // forward L w = b, then back L^T z = w, one thread per right-hand side
    for (int c = tid; c < nrhs; c += nt) {
        for (int i = 0; i < k; ++i) {
            double v = b[i * LD + c];
            for (int p = 0; p < i; ++p) v = fma(-s[i * LD + p], b[p * LD + c], v);
            b[i * LD + c] = v / s[i * LD + i];
        }
        for (int i = k - 1; i >= 0; --i) {
            double v = b[i * LD + c];
            for (int p = i + 1; p < k; ++p) v = fma(-s[p * LD + i], b[p * LD + c], v);
            b[i * LD + c] = v / s[i * LD + i];
        }
    }
    __syncthreads();
    for (int t = tid; t < k * nrhs; t += nt) Out[t] = b[(t / nrhs) * LD + t % nrhs];
}

__global__ void lu_solve_kernel(int defer, const double* __restrict__ G, const double* __restrict__ Rhs,
                                double* __restrict__ Out, int k, int nrhs, double sign, double tol,
                                DevStatus* st) {
    __shared__ double s[KM * LD];
    __shared__ double b[KM * LD];
    __shared__ int s_piv, s_fail;
    __shared__ double s_scale;
    if (st && st->halt) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < k * k; t += nt) s[(t / k) * LD + t % k] = G[t];
    for (int t = tid; t < k * nrhs; t += nt) b[(t / nrhs) * LD + t % nrhs] = sign * Rhs[t];
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int t = 0; t < k * k; ++t) m = fmax(m, fabs(G[t]));
        s_scale = m > 0.0 ? m : 2.2250738585072014e-308;
        s_fail = -1;
    }
    __syncthreads();
    for (int j = 0; j < k; ++j) {
        if (tid < 32) {  // warp 0: argmax |s[i][j]|, i >= j (first index on ties)
            double best = -1.0;
            int bi = j;
            for (int i = j + tid; i < k; i += 32) {
                const double v = fabs(s[i * LD + j]);
                if (v > best) { best = v; bi = i; }
            }
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, m);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (tid == 0) {
                s_piv = bi;
                if (!(best > tol * s_scale)) s_fail = j;
            }
        }
        __syncthreads();
        if (s_fail >= 0) {
            if (tid == 0 && st) {
                if (defer) st->pending_bd = s_fail + 1;
                else { st->breakdown_col = s_fail; st->halt = 1; }
            }
            return;
        }
        const int p = s_piv;
        if (p != j) {
            for (int c = tid; c < k; c += nt) { double t = s[j * LD + c]; s[j * LD + c] = s[p * LD + c]; s[p * LD + c] = t; }
            for (int c = tid; c < nrhs; c += nt) { double t = b[j * LD + c]; b[j * LD + c] = b[p * LD + c]; b[p * LD + c] = t; }
        }
        __syncthreads();
        const int m = k - j - 1;
        // eliminate below the pivot: row r -= f_r * row j (matrix part then rhs)
        for (int t = tid; t < m * (k - j + nrhs); t += nt) {
            const int r = j + 1 + t / (k - j + nrhs), c = t % (k - j + nrhs);
            const double f = s[r * LD + j] / s[j * LD + j];
            if (c < k - j) {
                if (c > 0) s[r * LD + j + c] = fma(-f, s[j * LD + j + c], s[r * LD + j + c]);
            } else {
                const int cc = c - (k - j);
                b[r * LD + cc] = fma(-f, b[j * LD + cc], b[r * LD + cc]);
            }
        }
        __syncthreads();
        for (int r = j + 1 + tid; r < k; r += nt) s[r * LD + j] = 0.0;
        __syncthreads();
    }
    for (int c = tid; c < nrhs; c += nt) {
        for (int i = k - 1; i >= 0; --i) {
            double v = b[i * LD + c];
            for (int q = i + 1; q < k; ++q) v = fma(-s[i * LD + q], b[q * LD + c], v);
            b[i * LD + c] = v / s[i * LD + i];
        }
    }
    __syncthreads();
    for (int t = tid; t < k * nrhs; t += nt) Out[t] = b[(t / nrhs) * LD + t % nrhs];
}

// CholQR factor: G = R^T R (R upper = L^T), Rinv = R^{-1}, Rprod = R * Rprev.
__global__ void chol_qr_kernel(const double* __restrict__ G, double* __restrict__ R, double* __restrict__ Rinv,
                               const double* __restrict__ Rprev, double* __restrict__ Rprod, int k, double tol,
                               DevStatus* st) {
    __shared__ double s[KM * LD];
    __shared__ double inv[KM * LD];
    if (st && st->halt) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < k * k; t += nt) s[(t / k) * LD + t % k] = G[t];
    __syncthreads();
    const int fail = chol_lower_inplace(s, k, tol);
    if (fail >= 0) {
        if (tid == 0 && st) { st->breakdown_col = fail; st->halt = 1; }
        return;
    }
    // R[i][c] = L[c][i] for c >= i.  Rinv: solve R Z = I, column c by thread c.
    for (int c = tid; c < k; c += nt) {
        for (int i = k - 1; i >= 0; --i) {
            double v = (i == c) ? 1.0 : 0.0;
            for (int q = i + 1; q <= c; ++q) v = fma(-s[q * LD + i], inv[q * LD + c], v);
            inv[i * LD + c] = (i <= c) ? v / s[i * LD + i] : 0.0;
        }
    }
    __syncthreads();
    for (int t = tid; t < k * k; t += nt) {
        const int i = t / k, c = t % k;
        if (R) R[t] = (c >= i) ? s[c * LD + i] : 0.0;
        Rinv[t] = (c >= i) ? inv[i * LD + c] : 0.0;
    }
    if (Rprev && Rprod) {
        for (int t = tid; t < k * k; t += nt) {
            const int i = t / k, c = t % k;
            double v = 0.0;
            for (int q = i; q < k; ++q) v = fma(s[q * LD + i], Rprev[q * k + c], v);  // R[i][q] = L[q][i]
            Rprod[t] = v;
        }
    }
}

__global__ void conv_check_kernel(const double* __restrict__ g, int gstride, int k, double rtol,
                                  int conv_mode, int init, DevStatus* st) {
    if (threadIdx.x != 0) return;
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

__global__ void omega_kernel(const double* ts, const double* tt, int k, int stride, DevStatus* st) {
    if (threadIdx.x != 0 || st->halt) return;
    double a = 0.0, b = 0.0;
    for (int c = 0; c < k; ++c) { a += ts[c * stride]; b += tt[c * stride]; }
    if (!(b > 0.0)) { st->breakdown_col = 0; st->halt = 1; return; }
    st->omega = a / b;
    st->neg_omega = -(a / b);
}

__global__ void copy_kernel(const double* src, double* dst, int n) {
    for (int t = threadIdx.x; t < n; t += blockDim.x) dst[t] = src[t];
}

__global__ void add_kernel(const double* a, const double* b, double* out, int n) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) out[t] = a[t] + b[t];
}

// ---------------------------------------------------------------- block GMRES LSQ
// Hcol: (j+2)k x k (row-major, ld k).  Qs: per block q a 2k x 2k orthogonal
// matrix (row-major).  g: (m+1)k x k (ld k).  Rtri: upper triangular (ld ldr).
__global__ void gmres_step_kernel(double* __restrict__ Hcol, int j, int k, double* __restrict__ Qs,
                                  double* __restrict__ Rtri, int ldr, double* __restrict__ g, double rtol,
                                  int conv_mode, DevStatus* st) {
    extern __shared__ double dyn[];
    __shared__ double s_alpha, s_vnorm2;
    if (st->halt) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int m2 = 2 * k;
    const int LH = k + 1, LQ = m2 + 1;
    double* h = dyn;                    // 2k x k working slice (ld LH)
    double* Q = h + m2 * LH;            // 2k x 2k (ld LQ)
    double* v = Q + m2 * LQ;            // 2k
    const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    // 1. apply Q_0^T .. Q_{j-1}^T to rows [qk, (q+2)k) of Hcol
    for (int q = 0; q < j; ++q) {
        double* hs = Hcol + (int64_t)q * k * k;
        const double* Qq = Qs + (int64_t)q * m2 * m2;
        for (int t = tid; t < m2 * k; t += nt) h[(t / k) * LH + t % k] = hs[t];
        __syncthreads();
        for (int t = tid; t < m2 * k; t += nt) {
            const int i = t / k, c = t % k;
            double acc = 0.0;
            for (int r = 0; r < m2; ++r) acc = fma(Qq[r * m2 + i], h[r * LH + c], acc);
            hs[t] = acc;
        }
        __syncthreads();
    }
    // rows [0, jk) are final entries of R's block column j
    for (int t = tid; t < j * k * k; t += nt) {
        const int i = t / k, c = t % k;
        Rtri[(int64_t)i * ldr + j * k + c] = Hcol[t];
    }
    // 2. Householder QR of the bottom slice S = Hcol[jk:(j+2)k] (2k x k), Q explicit
    double* hs = Hcol + (int64_t)j * k * k;
    for (int t = tid; t < m2 * k; t += nt) h[(t / k) * LH + t % k] = hs[t];
    for (int t = tid; t < m2 * m2; t += nt) Q[(t / m2) * LQ + t % m2] = (t / m2 == t % m2) ? 1.0 : 0.0;
    __syncthreads();
    for (int c = 0; c < k; ++c) {
        if (warp == 0) {
            double ss = 0.0;
            for (int i = c + lane; i < m2; i += 32) ss += h[i * LH + c] * h[i * LH + c];
            ss = warp_sum(ss);
            if (lane == 0) {
                const double x0 = h[c * LH + c];
                const double nrm = sqrt(ss);
                const double alpha = (x0 >= 0.0) ? -nrm : nrm;
                s_alpha = alpha;
                // v = x - alpha e1; |v|^2 = ss - 2 alpha x0 + alpha^2
                s_vnorm2 = ss - 2.0 * alpha * x0 + alpha * alpha;
            }
        }
        __syncthreads();
        const double alpha = s_alpha, vn2 = s_vnorm2;
        for (int i = tid; i < m2; i += nt) v[i] = (i < c) ? 0.0 : (h[i * LH + c] - (i == c ? alpha : 0.0));
        __syncthreads();
        if (vn2 > 0.0) {
            const double beta = 2.0 / vn2;
            // S[:, c'] -= beta v (v^T S[:, c']) for c' > c ; one warp per column
            for (int cc = c + 1 + warp; cc < k; cc += nwarps) {
                double d = 0.0;
                for (int i = c + lane; i < m2; i += 32) d += v[i] * h[i * LH + cc];
                d = warp_sum(d);
                for (int i = c + lane; i < m2; i += 32) h[i * LH + cc] = fma(-beta * d, v[i], h[i * LH + cc]);
            }
            // Q[r, :] -= beta (Q[r, :] v) v^T ; one warp per row
            for (int r = warp; r < m2; r += nwarps) {
                double d = 0.0;
                for (int i = c + lane; i < m2; i += 32) d += Q[r * LQ + i] * v[i];
                d = warp_sum(d);
                for (int i = c + lane; i < m2; i += 32) Q[r * LQ + i] = fma(-beta * d, v[i], Q[r * LQ + i]);
            }
        }
        __syncthreads();
        if (tid == 0) {
            h[c * LH + c] = vn2 > 0.0 ? alpha : h[c * LH + c];
            for (int i = c + 1; i < m2; ++i) h[i * LH + c] = 0.0;
        }
        __syncthreads();
    }
    // R_jj and Q_j
    for (int t = tid; t < k * k; t += nt) {
        const int i = t / k, c = t % k;
        Rtri[(int64_t)(j * k + i) * ldr + j * k + c] = (c >= i) ? h[i * LH + c] : 0.0;
    }
    double* Qj = Qs + (int64_t)j * m2 * m2;
    for (int t = tid; t < m2 * m2; t += nt) Qj[t] = Q[(t / m2) * LQ + t % m2];
    __syncthreads();
    // 3. g[jk:(j+2)k] = Q_j^T g[jk:(j+2)k]
    double* gs = g + (int64_t)j * k * k;
    for (int t = tid; t < m2 * k; t += nt) h[(t / k) * LH + t % k] = gs[t];
    __syncthreads();
    for (int t = tid; t < m2 * k; t += nt) {
        const int i = t / k, c = t % k;
        double acc = 0.0;
        for (int r = 0; r < m2; ++r) acc = fma(Q[r * LQ + i], h[r * LH + c], acc);
        gs[t] = acc;
    }
    __syncthreads();
    // 4. residual norms: rows (j+1)k .. (j+2)k of the rotated g
    if (tid == 0) {
        bool ok = true;
        for (int c = 0; c < k; ++c) {
            double ss = 0.0;
            for (int i = 0; i < k; ++i) { const double x = gs[(k + i) * k + c]; ss += x * x; }
            const double r0 = st->r0[c];
            const double rel = sqrt(ss) / (r0 > 0.0 ? r0 : 1.0);
            st->relres[c] = rel;
            if (conv_mode == BK_CONV_FIRST ? (c == 0 && !(rel <= rtol)) : !(rel <= rtol)) ok = false;
        }
        st->iter += 1;
        st->gm_steps = j + 1;
        if (ok) { st->converged = 1; st->halt = 1; }
    }
}

// Upper-triangular block back-substitution, column-oriented (parallel over the
// rows of the remaining right-hand side), one CTA.
__global__ void gmres_backsolve_kernel(const double* __restrict__ Rtri, int ldr, const double* __restrict__ g,
                                       double* __restrict__ y, int nk, int k) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int t = tid; t < nk * k; t += nt) y[t] = g[t];
    __syncthreads();
    for (int i = nk - 1; i >= 0; --i) {
        const double d = Rtri[(int64_t)i * ldr + i];
        for (int c = tid; c < k; c += nt) y[i * k + c] /= d;
        __syncthreads();
        for (int t = tid; t < i * k; t += nt) {
            const int r = t / k, c = t % k;
            y[t] = fma(-Rtri[(int64_t)r * ldr + i], y[i * k + c], y[t]);
        }
        __syncthreads();
    }
}

}  // namespace

// single-warp register versions (dense_warp.cu) are the default; BK_DENSE=cta
// selects the shared-memory CTA kernels above (A/B and cross-check)
void sdw_lu_solve(const double*, const double*, double*, int, int, double, double, DevStatus*, cudaStream_t, int,
                  double*, int*);
void sdw_chol_solve(const double*, const double*, double*, int, int, double, DevStatus*, cudaStream_t);
void sdw_chol_qr(const double*, double*, double*, const double*, double*, int, double, DevStatus*, cudaStream_t);

static bool dense_cta() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("BK_DENSE");
        v = (e && e[0] == 'c') ? 1 : 0;
    }
    return v == 1;
}

void sd_chol_solve(const double* G, const double* Rhs, double* Out, int k, int nrhs, double tol, DevStatus* st,
                   cudaStream_t s) {
    if (!dense_cta()) return sdw_chol_solve(G, Rhs, Out, k, nrhs, tol, st, s);
    BK_KERNEL(chol_solve_kernel<<<1, 256, 0, s>>>(G, Rhs, Out, k, nrhs, tol, st));
}
void sd_lu_solve(const double* G, const double* Rhs, double* Out, int k, int nrhs, double sign, double tol,
                 DevStatus* st, cudaStream_t s, int defer, double* LUo, int* pivo) {
    if (!dense_cta() || LUo) return sdw_lu_solve(G, Rhs, Out, k, nrhs, sign, tol, st, s, defer, LUo, pivo);
    BK_KERNEL(lu_solve_kernel<<<1, 256, 0, s>>>(defer, G, Rhs, Out, k, nrhs, sign, tol, st));
}
void sd_chol_qr(const double* G, double* R, double* Rinv, const double* Rprev, double* Rprod, int k, double tol,
                DevStatus* st, cudaStream_t s) {
    if (!dense_cta()) return sdw_chol_qr(G, R, Rinv, Rprev, Rprod, k, tol, st, s);
    BK_KERNEL(chol_qr_kernel<<<1, 256, 0, s>>>(G, R, Rinv, Rprev, Rprod, k, tol, st));
}
void sd_conv_check(const double* g, int gstride, int k, double rtol, int conv_mode, int init, DevStatus* st,
                   cudaStream_t s) {
    BK_KERNEL(conv_check_kernel<<<1, 32, 0, s>>>(g, gstride, k, rtol, conv_mode, init, st));
}
void sd_omega(const double* ts, const double* tt, int k, DevStatus* st, cudaStream_t s, int stride) {
    BK_KERNEL(omega_kernel<<<1, 32, 0, s>>>(ts, tt, k, stride, st));
}
void sd_copy(const double* src, double* dst, int n, cudaStream_t s) { BK_KERNEL(copy_kernel<<<1, 256, 0, s>>>(src, dst, n)); }
void sd_add(const double* a, const double* b, double* out, int n, cudaStream_t s) {
    BK_KERNEL(add_kernel<<<(n + 255) / 256 < 64 ? (n + 255) / 256 : 64, 256, 0, s>>>(a, b, out, n));
}
void sd_gmres_step(double* Hcol, int j, int k, double* Qs, double* Rtri, int ldr, double* g, double rtol,
                   int conv_mode, DevStatus* st, cudaStream_t s) {
    const size_t smem = (size_t)(2 * k * (k + 1) + 2 * k * (2 * k + 1) + 2 * k) * sizeof(double);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gmres_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr_set = true;
    }
    BK_KERNEL(gmres_step_kernel<<<1, 512, smem, s>>>(Hcol, j, k, Qs, Rtri, ldr, g, rtol, conv_mode, st));
}
void sd_gmres_backsolve(const double* Rtri, int ldr, const double* g, double* y, int nk, int k, cudaStream_t s) {
    BK_KERNEL(gmres_backsolve_kernel<<<1, 512, 0, s>>>(Rtri, ldr, g, y, nk, k));
}

}  // namespace bk
