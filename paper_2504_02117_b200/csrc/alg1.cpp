// alg1.cpp -- SURVEY.md §8(f) NEXT-3: Algorithm 1 "Block Krylov Time Stepping with
// Pipelining" (§2.2) on the nonlinear diffusion-reaction problem
// (R29-R31, oracle O10).  Host orchestration only: every N x w step is a
// library kernel (f / Jacobian assembly in nonlin.cu, block updates, Gram, the block
// Krylov solve of "solve JV = R").
//   window of w consecutive global stages g0 .. g0+w-1 (stage s: step s / m, index s % m);
//   R(Y) = M Y A1^T + F(T, Y) A2^T - B0                       (sign R30)
//   B0 = Hist Cb, Hist = [y^n, f_0, ..., f_{m-2}] (the current step's accepted stages)
//   per stage: Y <- shift(Y); loop: R <- R(Y); ||R_0|| < eps -> accept; else
//   J <- M/tau + a_kk Df(t_0, Y_0); solve J V = R; Y <- Y - V.
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstring>
#include <vector>

#include "bk_internal.h"

namespace bk {

namespace {
enum { WS_ALG1 = 112 };   // workspace slots WS_ALG1 .. WS_ALG1 + 9

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

int alg1_impl(bk_ctx* ctx, const bk_dr_problem* pb, int m, const double* Atab, int n_steps, int w, double eps,
              int max_newton, const bk_solve_opts* inner, double* traj, int64_t ldt, int* newton_its,
              bk_alg1_report* rep) {
    cudaStream_t st = ctx->stream;
    const int64_t nx = pb->nx, ny = pb->ny, nz = pb->nz, N = nx * ny * nz;
    const double h = 1.0 / (double)nx, mass = h * h * h, tau = pb->tau;
    memset(rep, 0, sizeof *rep);
    rep->status = BK_OK;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    // ---- Newton matrix: 7-point lattice pattern (ascending columns), values per iteration
    std::vector<int32_t> rp(N + 1), cols;
    cols.reserve(7 * N);
    rp[0] = 0;
    for (int64_t a = 0; a < N; ++a) {
        const int64_t ix = a % nx, iy = (a / nx) % ny, iz = a / (nx * ny);
        const int64_t off[7] = {-nx * ny, -nx, -1, 0, 1, nx, nx * ny};
        const bool has[7] = {iz > 0, iy > 0, ix > 0, true, ix < nx - 1, iy < ny - 1, iz < nz - 1};
        for (int d = 0; d < 7; ++d)
            if (has[d]) cols.push_back((int32_t)(a + off[d]));
        rp[a + 1] = (int32_t)cols.size();
    }
    std::vector<double> zeros(cols.size(), 0.0);
    bk_csr* J = nullptr;
    int r = bk_csr_create(ctx, &J, N, 0, N, rp.data(), cols.data(), zeros.data(), (int64_t)cols.size());
    if (r) return r;
    struct Guard {
        bk_csr* J;
        cudaEvent_t a, b;
        ~Guard() { bk_csr_destroy(J); cudaEventDestroy(a); cudaEventDestroy(b); }
    } guard{J, e0, e1};
    // ---- device buffers
    const int H = 1 + m;                                       // Hist columns
    const size_t vb = (size_t)N * w * sizeof(double);
    double* Y = (double*)ws_get(ctx, WS_ALG1, vb);
    double* Y2 = (double*)ws_get(ctx, WS_ALG1 + 1, vb);
    double* F = (double*)ws_get(ctx, WS_ALG1 + 2, vb);
    double* R = (double*)ws_get(ctx, WS_ALG1 + 3, vb);
    double* V = (double*)ws_get(ctx, WS_ALG1 + 4, vb);
    double* Hist = (double*)ws_get(ctx, WS_ALG1 + 5, (size_t)N * H * sizeof(double));
    double* gdev = (double*)ws_get(ctx, WS_ALG1 + 6, (size_t)N * sizeof(double));
    // small: C1 = mass A1^T (w x w), C2 = A2^T (w x w), Cb (H x w), S (w x w), sinT (w), G (1), bad flag
    const size_t sm_d = 5 * (size_t)w * w + (size_t)H * w + w + (size_t)w * w + 8;
    double* sm = (double*)ws_get(ctx, WS_ALG1 + 7, sm_d * sizeof(double));
    double *dC1 = sm, *dC2 = dC1 + w * w, *dCb = dC2 + w * w, *dS = dCb + H * w, *dsin = dS + 2 * w * w,
           *dG = dsin + w;
    int* dbad = reinterpret_cast<int*>(dG + w * w);
    double* hsm = (double*)ctx->h_pinned;                      // pinned staging (>= 64 KB)
    auto cu = [&](cudaError_t e, const char* what) { return cuda_check(ctx, e, what); };
    if ((r = cu(cudaMemcpyAsync(gdev, pb->g, N * sizeof(double), cudaMemcpyDefault, st), "alg1 g"))) return r;
    if ((r = cu(cudaMemsetAsync(dbad, 0, sizeof(int), st), "alg1 bad"))) return r;
    // Y = (y0, ..., y0); Hist[:, 0] = y0
    {
        std::vector<double> ones(w, 1.0);
        if ((r = cu(cudaMemcpyAsync(Hist, pb->y0, N * sizeof(double), cudaMemcpyDefault, st), "alg1 y0"))) return r;
        // Hist column 0 holds y0 contiguously for now -> spread: Y = y0 1^T via a k=1 -> w update
        if ((r = cu(cudaMemcpyAsync(V, pb->y0, N * sizeof(double), cudaMemcpyDefault, st), "alg1 y0"))) return r;
        if ((r = cu(cudaMemcpyAsync(dS, ones.data(), w * sizeof(double), cudaMemcpyHostToDevice, st), "alg1 ones")))
            return r;
        upd(ctx, N, w, Y, w, 0.0, nullptr, w, 1.0, V, 1, 1, dS);   // Y = y0 * ones(1 x w)
        upd(ctx, N, 1, Hist, H, 0.0, nullptr, H, 0.0, nullptr, 1, 0, nullptr, V, 1, 1.0);   // Hist[:,0] = y0
        if ((r = cu(cudaStreamSynchronize(st), "alg1 init"))) return r;
    }
    std::vector<double> A(Atab, Atab + m * m), c(m, 0.0);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) c[i] += A[i * m + j];
    bk_solve_opts o = *inner;
    o.x0_is_zero = 1;
    int naccept = 0;   // accepted stages of the current step (f values in Hist[:, 1 + j])
    const int total = n_steps * m;
    bool first = true;
    for (int g0 = 0; g0 < total; ++g0) {
        if (!first) {   // Y <- shift(Y) = Y S  (S[j][i] = 1 for j = min(i + 1, w - 1))
            std::vector<double> S(w * w, 0.0);
            for (int i = 0; i < w; ++i) S[std::min(i + 1, w - 1) * w + i] = 1.0;
            memcpy(hsm, S.data(), S.size() * sizeof(double));
            if ((r = cu(cudaMemcpyAsync(dS, hsm, S.size() * sizeof(double), cudaMemcpyHostToDevice, st), "shift")))
                return r;
            upd(ctx, N, w, Y2, w, 0.0, nullptr, w, 1.0, Y, w, w, dS);
            std::swap(Y, Y2);
            if ((r = cu(cudaStreamSynchronize(st), "shift sync"))) return r;   // hsm / dS reuse
        }
        first = false;
        const int n = g0 / m, ck = g0 % m;
        // window matrices (P:260-288 rows / columns g0 .. g0 + w - 1), B0 coefficients, stage times
        std::vector<double> hb(2 * w * w + H * w + w, 0.0);
        double *C1 = hb.data(), *C2 = C1 + w * w, *Cb = C2 + w * w, *sinT = Cb + H * w;
        for (int i = 0; i < w; ++i) {
            const int si = g0 + i, qi = si / m, ci = si % m;
            for (int j = 0; j < w; ++j) {
                const int sj = g0 + j, qj = sj / m, cj = sj % m;
                double a1 = (i == j) ? 1.0 / tau : 0.0;
                if (qi >= 1 && sj == qi * m - 1) a1 = -1.0 / tau;
                const double a2 = (qj == qi) ? A[ci * m + cj] : 0.0;
                C1[j * w + i] = mass * a1;   // C1 = mass A1^T: C1[j][i] = mass A1[i][j]
                C2[j * w + i] = a2;
            }
            if (qi == n) {   // B0_i = (1/tau) M y^n - sum_{accepted j} a_{c_i j} f_j
                Cb[0 * w + i] = mass / tau;
                for (int j = 0; j < naccept; ++j) Cb[(1 + j) * w + i] = -A[ci * m + j];
            }
            sinT[i] = std::sin(1.0 + (qi * tau + tau * c[ci]));
        }
        memcpy(hsm, hb.data(), hb.size() * sizeof(double));
        if ((r = cu(cudaMemcpyAsync(dC1, hsm, 2 * w * w * sizeof(double), cudaMemcpyHostToDevice, st), "alg1 C")))
            return r;
        if ((r = cu(cudaMemcpyAsync(dCb, hsm + 2 * w * w, H * w * sizeof(double), cudaMemcpyHostToDevice, st),
                    "alg1 Cb")))
            return r;
        if ((r = cu(cudaMemcpyAsync(dsin, hsm + 2 * w * w + H * w, w * sizeof(double), cudaMemcpyHostToDevice, st),
                    "alg1 sin")))
            return r;
        int it = 0;
        for (;; ++it) {
            // R = -Hist Cb + Y (mass A1^T) + F A2^T
            launch_dr_f(nx, ny, nz, h, Y, w, w, dsin, gdev, F, w, st);
            upd(ctx, N, w, R, w, 0.0, nullptr, w, -1.0, Hist, H, H, dCb);
            upd(ctx, N, w, R, w, 1.0, R, w, 1.0, Y, w, w, dC1);
            upd(ctx, N, w, R, w, 1.0, R, w, 1.0, F, w, w, dC2);
            if ((r = gram_dev(ctx, N, w, w, R, w, R, w, dG, false))) return r;   // column norms (diag)
            double* hg = hsm + 4096;
            if ((r = cu(cudaMemcpyAsync(hg, dG, w * w * sizeof(double), cudaMemcpyDeviceToHost, st), "alg1 norm")))
                return r;
            if ((r = cu(cudaStreamSynchronize(st), "alg1 sync"))) return r;
            const double nr0 = std::sqrt(std::max(hg[0], 0.0));
            if (nr0 < eps) break;                                           // lines 6-9
            if (it == max_newton) {
                rep->status = BK_NOT_CONVERGED;
                rep->failed_stage = g0;
                rep->last_norm = nr0;
                cudaEventRecord(e1, st);
                cudaStreamSynchronize(st);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                rep->t_total_ms = ms;
                return BK_NOT_CONVERGED;
            }
            // J = M/tau + a_kk Df(t_0, Y_0) (line 10); solve J V = R (line 11); Y -= V (line 12)
            launch_dr_jac(nx, ny, nz, h, Y, w, mass / tau, A[ck * m + ck], J->d_rp, J->d_col, J->d_val, dbad, st);
            launch_extract_diag_inv(N, 0, J->d_rp, J->d_col, J->d_val, J->d_dinv, st);
            if ((r = cu(cudaGetLastError(), "alg1 jacobian"))) return r;
            // columns scaled to unit norm before the block solve (V = J^-1 R is column-wise
            // linear): near convergence ||R_0|| << ||R_i|| and the block CholQR / Cholesky
            // would report breakdown on the relative pivot (R6, R31)
            double* hd = hsm + 4096 + 1024;
            for (int i = 0; i < 2 * w * w; ++i) hd[i] = 0.0;
            for (int i = 0; i < w; ++i) {
                const double nrm = std::sqrt(std::max(hg[i * w + i], 0.0));
                hd[i * w + i] = nrm > 0.0 ? 1.0 / nrm : 1.0;
                hd[w * w + i * w + i] = nrm > 0.0 ? nrm : 1.0;
            }
            if ((r = cu(cudaMemcpyAsync(dS, hd, 2 * w * w * sizeof(double), cudaMemcpyHostToDevice, st), "alg1 D")))
                return r;
            upd(ctx, N, w, Y2, w, 0.0, nullptr, w, 1.0, R, w, w, dS);        // Rs = R D^-1
            bk_solve_report sr;
            r = solve_impl(ctx, J, w, Y2, w, V, w, &o, &sr);
            if (r == BK_ERR_CUDA || r == BK_ERR_NCCL || r == BK_ERR_OOM || r == BK_ERR_ARG) return r;
            rep->inner_iterations_total += sr.iterations;
            rep->newton_iterations_total += 1;
            if (sr.status == BK_BREAKDOWN) {
                // rank-deficient block (e.g. the first iterate Y = (y0, ..., y0): every column's
                // residual lies in span{K(y0) y0, g}); the block methods do not deflate (R6),
                // so the columns are solved one by one (R31)
                rep->inner_breakdowns += 1;
                for (int i = 0; i < w; ++i) {
                    r = solve_impl(ctx, J, 1, Y2 + i, w, V + i, w, &o, &sr);
                    if (r == BK_ERR_CUDA || r == BK_ERR_NCCL || r == BK_ERR_OOM || r == BK_ERR_ARG) return r;
                    rep->inner_iterations_total += sr.iterations;
                }
            }
            upd(ctx, N, w, Y, w, 1.0, Y, w, -1.0, V, w, w, dS + w * w);     // Y -= Vs D
        }
        if (newton_its) newton_its[g0] = it;
        // accept column 0: stiffly accurate -> y^{n+1} = last stage, else keep f of the stage
        if (ck == m - 1) {
            upd(ctx, N, 1, Hist, H, 0.0, nullptr, H, 0.0, nullptr, 1, 0, nullptr, Y, w, 1.0);   // Hist[:,0] = Y_0
            if (traj) {
                if (is_device_ptr(traj)) {
                    upd(ctx, N, 1, traj + n, ldt, 0.0, nullptr, ldt, 0.0, nullptr, 1, 0, nullptr, Y, w, 1.0);
                } else {   // contiguous staging column, then one D2H copy into the strided host column
                    upd(ctx, N, 1, V, 1, 0.0, nullptr, 1, 0.0, nullptr, 1, 0, nullptr, Y, w, 1.0);
                    if ((r = cu(cudaMemcpy2DAsync(traj + n, ldt * sizeof(double), V, sizeof(double), sizeof(double),
                                                  N, cudaMemcpyDeviceToHost, st),
                                "alg1 traj")))
                        return r;
                }
            }
            naccept = 0;
        } else {
            upd(ctx, N, 1, Hist + 1 + ck, H, 0.0, nullptr, H, 0.0, nullptr, 1, 0, nullptr, F, w, 1.0);
            naccept = ck + 1;
        }
        if ((r = cu(cudaGetLastError(), "alg1 accept"))) return r;
        rep->stages_accepted += 1;
    }
    int hbad = 0;
    if ((r = cu(cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st), "alg1 bad"))) return r;
    cudaEventRecord(e1, st);
    if ((r = cu(cudaStreamSynchronize(st), "alg1 end"))) return r;
    if (hbad) return set_error(ctx, BK_ERR_ARG, "alg1: Jacobian pattern mismatch (internal)");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    rep->t_total_ms = ms;
    return BK_OK;
}

}  // namespace bk
