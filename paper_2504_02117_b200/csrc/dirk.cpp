// dirk.cpp -- SURVEY.md §8(f) NEXT-1: a window of s time steps x m stages of a
// stiffly accurate DIRK method as ONE matrix equation (§2.1,
// eq. general-system-time-steps, window matrices P:260-288),
//     M Y A1^T + K Y A2^T = B A2^T + B0,      M = mass * I,
// solved by the splitting fixed point (eq. matrix-splitting and
// matrix-fixed-point-equation), beta = A2[0][0]:
//     (M/tau + beta K) Y^j = -M Y^{j-1} (A1 - I/tau)^T - K Y^{j-1} (A2 - beta I)^T + B A2^T + B0.
// Host orchestration only: every N x k step is a library kernel (block update,
// coupled apply, block Krylov solve, Gram).  The right-hand side of one outer
// iteration costs one DMMA update pass and one coupled apply (the k x k
// coupling applied in the apply's epilogue).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "bk_internal.h"

namespace bk {

namespace {
enum { WS_DIRK = 96 };   // workspace slots WS_DIRK .. WS_DIRK + 7 (the solver uses WS_SOLVE_BASE + i < 96)

void upd(bk_ctx* ctx, int64_t n, int k, double* out, int64_t ldo, double a, const double* Xin, int64_t ldxin,
         double s, const double* P, int64_t ldp, int kp, const double* C, const double* W = nullptr,
         int64_t ldw = 0, double w = 0.0) {
    UpdArgs u{};
    u.n = n; u.kp = kp; u.k = k;
    u.a = a; u.Xin = Xin; u.ldxin = ldxin;
    u.s = s; u.P = P; u.ldp = ldp; u.C = C;
    u.W = W; u.ldw = ldw; u.w_host = w; u.w_dev = nullptr;
    u.out = out; u.ldo = ldo;
    u.halt = nullptr;
    launch_update(u, ctx->stream);
}
}  // namespace

int dirk_impl(bk_ctx* ctx, const bk_csr* L, const bk_csr* K, double mass, double tau, int k, const double* A1h,
              const double* A2h, const double* B, const double* B0, int64_t ldb, double* Y, int64_t ldy,
              int max_outer, double outer_tol, const bk_solve_opts* inner, bk_dirk_report* rep, bool correction) {
    cudaStream_t st = ctx->stream;
    const int64_t n = L->n_local;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    // k x k right multipliers (row-major): C1 = -mass (A1 - I/tau)^T, C2 = (A2 - beta I)^T, A2^T
    const double beta = A2h[0];
    std::vector<double> h(3 * (size_t)k * k);
    double *C1 = h.data(), *C2 = C1 + k * k, *A2T = C2 + k * k;
    for (int r = 0; r < k; ++r)
        for (int c = 0; c < k; ++c) {
            C1[r * k + c] = -mass * (A1h[c * k + r] - (r == c ? 1.0 / tau : 0.0));
            C2[r * k + c] = A2h[c * k + r] - (r == c ? beta : 0.0);
            A2T[r * k + c] = A2h[c * k + r];
        }
    double* dsm = (double*)ws_get(ctx, WS_DIRK, h.size() * sizeof(double) + 4 * 32 * 32 * sizeof(double));
    double *dC1 = dsm, *dC2 = dC1 + k * k, *dA2T = dC2 + k * k, *G = dsm + h.size();
    int r = cuda_check(ctx, cudaMemcpyAsync(dsm, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, st),
                       "dirk coefficients");
    if (r) return r;
    const size_t vb = (size_t)(n > 0 ? n : 1) * k * sizeof(double);
    double* R0 = (double*)ws_get(ctx, WS_DIRK + 1, vb);
    double* Rhs = (double*)ws_get(ctx, WS_DIRK + 2, vb);
    double* Yp = (double*)ws_get(ctx, WS_DIRK + 3, vb);
    double* D = (double*)ws_get(ctx, WS_DIRK + 4, vb);
    double* Ds = (double*)ws_get(ctx, WS_DIRK + 5, vb);
    double* hsm = (double*)ctx->h_pinned + 8192;   // pinned staging for the column scales
    // R0 = B0 + B A2^T (fixed part of every right-hand side)
    if (n > 0) {
        upd(ctx, n, k, R0, k, 1.0, B0, ldb, 1.0, B, ldb, k, dA2T);
        r = cuda_check(ctx, cudaGetLastError(), "dirk R0");
        if (r) return r;
    }
    // inner solves start from zero: with a warm start the columns the strictly lower
    // triangular coupling has already made exact have a zero residual, and the
    // block method breaks down on the rank-deficient residual block (no deflation,
    // DESIGN.md R6 / R26)
    bk_solve_opts o = *inner;
    o.x0_is_zero = 1;
    memset(rep, 0, sizeof *rep);
    rep->status = BK_OK;
    double change = 0.0, ff0 = 0.0;
    int j = 0;
    for (; j < max_outer && correction; ++j) {
        // defect correction (loose inner tolerance, the outer iterations refresh the
        // right-hand side): F = Rhs(Y) - L Y; L D = F (x0 = 0, inner rtol relative to F); Y += D.
        // Columns of F are scaled to unit norm first (converged stages have tiny defects; the
        // block methods do not deflate, R6); a block breakdown falls back to column-wise solves.
        if (n > 0) {
            upd(ctx, n, k, Rhs, k, 1.0, R0, k, 1.0, Y, ldy, k, dC1);
            r = cuda_check(ctx, cudaGetLastError(), "dirk rhs");
            if (r) return r;
        }
        r = spmm_dev(ctx, K, k, Y, ldy, dC2, k, -1.0, 1.0, Rhs, k);
        if (!r) r = spmm_dev(ctx, L, k, Y, ldy, nullptr, k, -1.0, 1.0, Rhs, k);   // F = Rhs - L Y
        if (!r) r = gram_dev(ctx, n, k, k, Rhs, k, Rhs, k, G, ctx->nranks > 1);
        if (!r) r = gram_dev(ctx, n, k, k, Y, ldy, Y, ldy, G + k * k, ctx->nranks > 1);
        if (r) return r;
        if ((r = cuda_check(ctx, cudaMemcpyAsync(hsm, G, 2 * (size_t)k * k * sizeof(double), cudaMemcpyDeviceToHost,
                                                 st), "dirk defect")))
            return r;
        if ((r = cuda_check(ctx, cudaStreamSynchronize(st), "dirk sync"))) return r;
        double ff = 0.0, yy = 0.0;
        std::vector<double> sc(2 * (size_t)k * k, 0.0);
        for (int c = 0; c < k; ++c) {
            const double fc = std::sqrt(std::max(hsm[c * k + c], 0.0));
            ff += hsm[c * k + c];
            yy += hsm[k * k + c * k + c];
            sc[c * k + c] = fc > 0.0 ? 1.0 / fc : 1.0;
            sc[k * k + c * k + c] = fc > 0.0 ? fc : 0.0;
        }
        // outer test on the defect reduction ||F^j||_F / ||F^0||_F (before solving)
        if (j == 0) ff0 = ff;
        change = ff0 > 0.0 ? std::sqrt(ff / ff0) : 0.0;
        if (j > 0 && outer_tol > 0.0 && change <= outer_tol) break;
        double* dsc = G + 2 * k * k;
        if ((r = cuda_check(ctx, cudaMemcpyAsync(dsc, sc.data(), sc.size() * sizeof(double), cudaMemcpyHostToDevice,
                                                 st), "dirk scales")))
            return r;
        if (n > 0) upd(ctx, n, k, Ds, k, 0.0, nullptr, k, 1.0, Rhs, k, k, dsc);   // Fs = F S^-1
        bk_solve_report sr;
        r = solve_impl(ctx, L, k, Ds, k, D, k, &o, &sr);
        if (r == BK_ERR_CUDA || r == BK_ERR_NCCL || r == BK_ERR_OOM || r == BK_ERR_ARG) return r;
        rep->inner_iterations_total += sr.iterations;
        rep->last_inner_status = sr.status;
        if (sr.status == BK_BREAKDOWN) {   // rank-deficient defect block: one column at a time
            for (int c = 0; c < k; ++c) {
                r = solve_impl(ctx, L, 1, Ds + c, k, D + c, k, &o, &sr);
                if (r == BK_ERR_CUDA || r == BK_ERR_NCCL || r == BK_ERR_OOM || r == BK_ERR_ARG) return r;
                rep->inner_iterations_total += sr.iterations;
                if (sr.status == BK_BREAKDOWN) { rep->status = BK_BREAKDOWN; break; }
            }
            if (rep->status == BK_BREAKDOWN) { ++j; break; }
        }
        if (n > 0) upd(ctx, n, k, Y, ldy, 1.0, Y, ldy, 1.0, D, k, k, dsc + k * k);   // Y += D S
        (void)yy;
    }
    for (; j < max_outer && !correction; ++j) {
        if (n > 0) {
            // Rhs = R0 + Y C1 - K Y C2   (one update pass + one coupled apply)
            upd(ctx, n, k, Rhs, k, 1.0, R0, k, 1.0, Y, ldy, k, dC1);
            r = cuda_check(ctx, cudaGetLastError(), "dirk rhs");
            if (r) return r;
        }
        r = spmm_dev(ctx, K, k, Y, ldy, dC2, k, -1.0, 1.0, Rhs, k);
        if (r) return r;
        if (n > 0) {   // Y^{j-1} kept for the change test (the solve overwrites Y)
            r = cuda_check(ctx,
                           ldy == k ? cudaMemcpyAsync(Yp, Y, vb, cudaMemcpyDeviceToDevice, st)
                                    : cudaMemcpy2DAsync(Yp, k * sizeof(double), Y, ldy * sizeof(double),
                                                        k * sizeof(double), n, cudaMemcpyDeviceToDevice, st),
                           "dirk copy");
            if (r) return r;
        }
        bk_solve_report sr;
        r = solve_impl(ctx, L, k, Rhs, k, Y, ldy, &o, &sr);
        if (r == BK_ERR_CUDA || r == BK_ERR_NCCL || r == BK_ERR_OOM || r == BK_ERR_ARG) return r;
        rep->inner_iterations_total += sr.iterations;
        rep->last_inner_status = sr.status;
        if (sr.status == BK_BREAKDOWN) {
            rep->status = BK_BREAKDOWN;
            ++j;
            break;
        }
        if (sr.status == BK_NOT_CONVERGED) rep->status = BK_NOT_CONVERGED;
        // relative change ||Y^j - Y^{j-1}||_F / ||Y^j||_F (Gram traces, summed over ranks)
        if (n > 0) upd(ctx, n, k, D, k, 1.0, Y, ldy, 0.0, nullptr, k, 0, nullptr, Yp, k, -1.0);
        r = gram_dev(ctx, n, k, k, D, k, D, k, G, ctx->nranks > 1);
        if (!r) r = gram_dev(ctx, n, k, k, Y, ldy, Y, ldy, G + k * k, ctx->nranks > 1);
        if (r) return r;
        std::vector<double> hg(2 * (size_t)k * k);
        r = cuda_check(ctx, cudaMemcpyAsync(hg.data(), G, hg.size() * sizeof(double), cudaMemcpyDeviceToHost, st),
                       "dirk change");
        if (!r) r = cuda_check(ctx, cudaStreamSynchronize(st), "dirk sync");
        if (r) return r;
        double dd = 0.0, yy = 0.0;
        for (int c = 0; c < k; ++c) {
            dd += hg[c * k + c];
            yy += hg[k * k + c * k + c];
        }
        change = yy > 0.0 ? std::sqrt(dd / yy) : std::sqrt(dd);
        if (outer_tol > 0.0 && change <= outer_tol) {
            ++j;
            break;
        }
    }
    rep->outer_iterations = j;
    rep->last_change = change;
    cudaEventRecord(e1, st);
    r = cuda_check(ctx, cudaStreamSynchronize(st), "dirk end");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    rep->t_total_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (r) return r;
    return rep->status;
}

}  // namespace bk

// ---------------------------------------------------------------- window matrices (host only)
// PAPER.md §2.1: s consecutive steps of a stiffly accurate DIRK tableau A (m x m) as one matrix
// equation (window matrices P:260-288, R24); an explicit first stage (a_11 = 0) is
// eliminated first: its row goes, its column a_{i1} couples the remaining stages to
// y^(n,1) = y^n -- for step q >= 1 that is the last stage of step q-1 (an A2 entry at the
// position of A1's -1/tau), for step 0 a B0 term (bk_dirk_b0).
namespace {
bool dirk_tableau_ok(int m, const double* A, bool* expl) {
    if (m < 1 || !A) return false;
    for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j)
            if (A[i * m + j] != 0.0) return false;   // diagonally implicit: lower triangular
    *expl = A[0] == 0.0;
    if (*expl && m == 1) return false;
    for (int i = *expl ? 1 : 0; i < m; ++i)
        if (A[i * m + i] == 0.0) return false;        // only the first stage may be explicit
    return true;
}
}  // namespace

extern "C" int bk_dirk_window(int m, const double* A, int s, double tau, int* k_out, double* A1, double* A2,
                              double* a_elim) {
    bool expl = false;
    if (!dirk_tableau_ok(m, A, &expl) || s < 1 || !(tau > 0.0) || !k_out || !A1 || !A2) return BK_ERR_ARG;
    const int o = expl ? 1 : 0, mi = m - o, k = s * mi;
    if (k > BK_MAX_K) return BK_ERR_ARG;
    std::memset(A1, 0, sizeof(double) * k * k);
    std::memset(A2, 0, sizeof(double) * k * k);
    for (int q = 0; q < s; ++q)
        for (int i = 0; i < mi; ++i) {
            const int row = q * mi + i;
            A1[row * k + row] = 1.0 / tau;
            for (int j = 0; j <= i; ++j) A2[row * k + q * mi + j] = A[(i + o) * m + (j + o)];
            if (q >= 1) {
                A1[row * k + q * mi - 1] = -1.0 / tau;
                if (expl) A2[row * k + q * mi - 1] = A[(i + 1) * m];
            }
        }
    if (a_elim)
        for (int i = 0; i < mi; ++i) a_elim[i] = expl ? A[(i + 1) * m] : 0.0;
    *k_out = k;
    return BK_OK;
}

namespace bk {
// B0 of the window (device): columns i < mi = (mass/tau) y^n + a_{i1} (b^n - K y^n) (the second
// term only for an eliminated explicit first stage), the other columns 0.  P:282-285.
int dirk_b0_impl(bk_ctx* ctx, const bk_csr* K, double mass, double tau, int m, const double* A, int s,
                 const double* yn, const double* bn, double* B0, int64_t ldb, double* scratch) {
    bool expl = false;
    dirk_tableau_ok(m, A, &expl);
    const int mi = expl ? m - 1 : m, k = s * mi;
    const int64_t n = K->n_local;
    cudaStream_t st = ctx->stream;
    int r = cuda_check(ctx, cudaMemset2DAsync(B0, ldb * sizeof(double), 0, k * sizeof(double), n, st), "dirk b0");
    if (r || n == 0) return r;
    // k x k coefficient rows (device): c_y = (mass / tau, ...), c_e = (a_21, ..., a_m1)
    std::vector<double> h(2 * mi);
    for (int i = 0; i < mi; ++i) {
        h[i] = mass / tau;
        h[mi + i] = expl ? A[(i + 1) * m] : 0.0;
    }
    double* dc = scratch + n;   // scratch: n doubles (K y^n) + 2 mi coefficients
    r = cuda_check(ctx, cudaMemcpyAsync(dc, h.data(), sizeof(double) * 2 * mi, cudaMemcpyHostToDevice, st), "dirk b0");
    if (r) return r;
    upd(ctx, n, mi, B0, ldb, 0.0, nullptr, 0, 1.0, yn, 1, 1, dc);            // (mass / tau) y^n
    if (expl) {
        r = spmm_dev(ctx, K, 1, yn, 1, nullptr, 1, 1.0, 0.0, scratch, 1);    // K y^n
        if (r) return r;
        if (bn) upd(ctx, n, mi, B0, ldb, 1.0, B0, ldb, 1.0, bn, 1, 1, dc + mi);
        upd(ctx, n, mi, B0, ldb, 1.0, B0, ldb, -1.0, scratch, 1, 1, dc + mi);
    }
    return cuda_check(ctx, cudaGetLastError(), "dirk b0");
}
}  // namespace bk

