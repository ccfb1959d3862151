// solve.cpp -- a6: block Krylov drivers (block CG, block GMRES(m), block BiCGStab).
//
// Host code that only ENQUEUES kernels on the ctx stream: the N x k work is
// bspmm / gram / update (spmm.cu, blas.cu), the k x k work runs in one-CTA
// kernels (dense.cu), and the convergence/breakdown state lives in a device
// DevStatus that the host polls every `check_every` iterations.  Kernels after
// a halt (convergence or breakdown) are no-ops, so X always holds the last
// valid iterate.  The algorithms follow DESIGN.md §3 readings O4-O6 step by
// step (the same steps as oracle/, written independently).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "bk_internal.h"

namespace bk {

// ---------------------------------------------------------------- NEXT-4 preconditioners (oracle O9)
void cheb_bounds(const bk_csr* A, const bk_solve_opts* o, double* lmin, double* lmax) {
    *lmax = o->cheb_lmax > 0.0 ? o->cheb_lmax : A->gersh;
    *lmin = o->cheb_lmin > 0.0 ? o->cheb_lmin : *lmax / 30.0;
}

bool cheb_opts_ok(const bk_csr* A, const bk_solve_opts* o) {
    double lo, hi;
    cheb_bounds(A, o, &lo, &hi);
    return o->cheb_steps >= 1 && lo > 0.0 && hi > lo && std::isfinite(hi);
}

namespace {
// Z = M^-1 R.  CHEBYSHEV (Saad Alg. 12.1 with the Jacobi splitting, the steps of O9):
//   d_0 = D^-1 R / theta, Z = d_0;  j = 1 .. steps-1: rho_j = 1/(2 sigma - rho_{j-1}),
//   d_j = rho_j rho_{j-1} d_{j-1} + (2 rho_j/delta) D^-1 (R - A Z), Z += d_j
// one apply + one fused elementwise pass (cheb_step_kernel) per step.  W, AZ: n x k scratch.
int prec_core(bk_ctx* ctx, const bk_csr* A, int k, const bk_solve_opts* o, const double* R, int64_t ldr,
              double* Z, int64_t ldz, double* W, double* AZ, int64_t* n_spmm) {
    const int64_t n = A->n_local;
    cudaStream_t st = ctx->stream;
    if (o->precond == BK_PRECOND_NONE) {
        if (n == 0) return BK_OK;
        return cuda_check(ctx,
                          cudaMemcpy2DAsync(Z, ldz * sizeof(double), R, ldr * sizeof(double), k * sizeof(double), n,
                                            cudaMemcpyDeviceToDevice, st),
                          "precond copy");
    }
    if (o->precond == BK_PRECOND_JACOBI) {
        launch_row_scale(n, k, A->d_dinv, R, ldr, Z, ldz, st);
        return cuda_check(ctx, cudaGetLastError(), "jacobi");
    }
    double lmin, lmax;
    cheb_bounds(A, o, &lmin, &lmax);
    const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma = theta / delta;
    double rho = 1.0 / sigma;
    launch_cheb_step(n, k, R, ldr, nullptr, A->d_dinv, W, Z, ldz, 0.0, 1.0 / theta, st);
    int r = cuda_check(ctx, cudaGetLastError(), "cheb_step");
    for (int j = 1; j < o->cheb_steps && !r; ++j) {
        const double rho_n = 1.0 / (2.0 * sigma - rho);
        r = spmm_dev(ctx, A, k, Z, ldz, nullptr, k, 1.0, 0.0, AZ, k);
        if (r) break;
        if (n_spmm) ++*n_spmm;
        launch_cheb_step(n, k, R, ldr, AZ, A->d_dinv, W, Z, ldz, rho_n * rho, 2.0 * rho_n / delta, st);
        r = cuda_check(ctx, cudaGetLastError(), "cheb_step");
        rho = rho_n;
    }
    return r;
}
}  // namespace

int precond_apply_impl(bk_ctx* ctx, const bk_csr* A, int k, const bk_solve_opts* o, const double* R, int64_t ldr,
                       double* Z, int64_t ldz) {
    enum { WS_PREC = 104 };
    const size_t vb = (size_t)std::max<int64_t>(A->n_local, 1) * k * sizeof(double);
    double* W = o->precond == BK_PRECOND_CHEBYSHEV ? (double*)ws_get(ctx, WS_PREC, vb) : nullptr;
    double* AZ = o->precond == BK_PRECOND_CHEBYSHEV ? (double*)ws_get(ctx, WS_PREC + 1, vb) : nullptr;
    return prec_core(ctx, A, k, o, R, ldr, Z, ldz, W, AZ, nullptr);
}

namespace {

struct Solver {
    bk_ctx* ctx;
    const bk_csr* A;
    int64_t n;
    int k;
    const bk_solve_opts* o;
    bk_solve_report* rep;
    cudaStream_t st;
    DevStatus* ds = nullptr;
    DevStatus* hs = nullptr;   // pinned readback
    int slot = WS_SOLVE_BASE;
    bool allred;
    // opts.timing: (start, end) event index pairs per kernel class, events from ctx->tev
    std::vector<int> tcls;
    int tnext = 0;
    cudaEvent_t tev(int i) {
        while ((int)ctx->tev.size() <= i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ctx->tev.push_back(e);
        }
        return ctx->tev[i];
    }
    void tb() {
        if (o->timing) cudaEventRecord(tev(tnext), st);
    }
    void te(int cls) {
        if (!o->timing) return;
        cudaEventRecord(tev(tnext + 1), st);
        tnext += 2;
        tcls.push_back(cls);
    }
    void tsum() {   // after the stream is synchronized
        for (size_t i = 0; i < tcls.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ctx->tev[2 * i], ctx->tev[2 * i + 1]);
            rep->t_class_ms[tcls[i]] += ms;
            rep->n_class[tcls[i]] += 1;
        }
    }

    double* vec(int ld_cols = 0) {
        const int cols = ld_cols ? ld_cols : k;
        return (double*)ws_get(ctx, slot++, (size_t)std::max<int64_t>(n, 1) * cols * sizeof(double));
    }
    double* small(size_t doubles) { return (double*)ws_get(ctx, slot++, doubles * sizeof(double)); }

    int init_status() {
        ds = (DevStatus*)ws_get(ctx, slot++, sizeof(DevStatus));
        DevStatus h;
        memset(&h, 0, sizeof h);
        h.breakdown_col = -1;
        DevStatus* pin = (DevStatus*)ctx->h_pinned;
        hs = (DevStatus*)((char*)ctx->h_pinned + 4096);
        if (!pin) return set_error(ctx, BK_ERR_OOM, "no pinned staging");
        *pin = h;
        return cuda_check(ctx, cudaMemcpyAsync(ds, pin, sizeof h, cudaMemcpyHostToDevice, st), "status init");
    }
    int poll() {
        int r = cuda_check(ctx, cudaMemcpyAsync(hs, ds, sizeof(DevStatus), cudaMemcpyDeviceToHost, st), "status poll");
        if (r) return r;
        return cuda_check(ctx, cudaStreamSynchronize(st), "status sync");
    }
    int launched(const char* w) { return cuda_check(ctx, cudaGetLastError(), w); }
    // Z = M^-1 R (JACOBI / CHEBYSHEV; W, AZ scratch for CHEBYSHEV)
    double *pw = nullptr, *paz = nullptr;
    int prec(const double* R, double* Z) {
        if (o->precond == BK_PRECOND_CHEBYSHEV && !pw) {
            pw = vec();
            paz = vec();
        }
        if (o->precond == BK_PRECOND_JACOBI) ab(2 * vb() + 8 * n);
        if (o->precond == BK_PRECOND_CHEBYSHEV)
            ab(3 * vb() + 8 * n + (int64_t)(o->cheb_steps - 1) * (spmm_b(false) + 7 * vb() + 8 * n));
        tb();
        const int r = prec_core(ctx, A, k, o, R, k, Z, k, pw, paz, &rep->n_spmm);
        te(BK_K_UPDATE);
        return r;
    }

    // Runs body() (one iteration) until max_iters or a halt, polling every check_every
    // iterations.  opts.use_graphs (one rank, no timing): after `period` eager iterations
    // (buffers allocated, kernel attributes set), `period` iterations are captured once into
    // a CUDA graph and replayed -- their kernel arguments are fixed (period 2 where the body
    // swaps two k x k buffers) and every update after a halt is a no-op, so replays past
    // convergence leave X unchanged.
    template <class F>
    int iterate(int period, F&& body) {
        const int maxit = o->max_iters, ce = o->check_every;
        bool graphs = o->use_graphs && !allred && !o->timing && n > 0;
        cudaGraphExec_t exec = nullptr;
        int64_t dl = 0, dsp = 0, dgr = 0, dup = 0, dsm = 0, dab = 0;   // per replay: launches, counters
        auto due = [&](int done) { return done % ce == 0 || done == maxit; };
        int it = 0, r = 0;
        while (it < maxit) {
            if (graphs && !exec && it >= period && maxit - it >= period) {
                const int64_t l0 = g_launches.load(), s0 = rep->n_spmm, g0 = rep->n_gram, u0 = rep->n_update,
                              m0 = rep->n_small, b0 = rep->alg_bytes;
                cudaGraph_t gph = nullptr;
                // capture on a private non-blocking stream (the ctx stream may be the legacy
                // default stream, which cannot be captured); replays go to the ctx stream
                if (!ctx->cap_stream) cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking);
                cudaStream_t keep = st;
                st = ctx->stream = ctx->cap_stream;
                bool ok = st && cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) == cudaSuccess;
                for (int q = 0; ok && q < period; ++q) ok = body() == 0;
                ok = (cudaStreamEndCapture(st, &gph) == cudaSuccess) && ok && gph;
                st = ctx->stream = keep;
                ok = ok && cudaGraphInstantiate(&exec, gph, 0) == cudaSuccess;
                if (gph) cudaGraphDestroy(gph);
                cudaGetLastError();
                dl = g_launches.load() - l0;   // captured, not launched yet
                g_launches -= dl;
                dsp = rep->n_spmm - s0; dgr = rep->n_gram - g0; dup = rep->n_update - u0; dsm = rep->n_small - m0;
                dab = rep->alg_bytes - b0;
                rep->n_spmm = s0; rep->n_gram = g0; rep->n_update = u0; rep->n_small = m0; rep->alg_bytes = b0;
                if (!ok) {   // fall back to eager launches
                    if (exec) cudaGraphExecDestroy(exec);
                    exec = nullptr;
                    graphs = false;
                    ctx->last_error.clear();
                    continue;
                }
            }
            if (exec && maxit - it >= period) {
                if ((r = cuda_check(ctx, cudaGraphLaunch(exec, st), "graph launch"))) break;
                rep->n_spmm += dsp; rep->n_gram += dgr; rep->n_update += dup; rep->n_small += dsm;
                rep->alg_bytes += dab;
                g_launches += dl;
                bool p = false;
                for (int q = 1; q <= period; ++q) p = p || due(it + q);
                it += period;
                if (p) {
                    if ((r = poll())) break;
                    if (hs->halt) break;
                }
                continue;
            }
            if ((r = body())) break;
            ++it;
            if (due(it)) {
                if ((r = poll())) break;
                if (hs->halt) break;
            }
        }
        if (exec) cudaGraphExecDestroy(exec);
        return r;
    }

    // algorithmic bytes of the passes this solve enqueues -> rep->alg_bytes
    int64_t vb() const { return 8 * n * k; }
    int64_t spmm_b(bool beta) const {
        return 12 * A->nnz + 4 * (n + 1) + 8 * (int64_t)k * (n + A->n_ghost) + vb() * (beta ? 2 : 1);
    }
    void ab(int64_t b) { rep->alg_bytes += b; }
    int spmm(const double* X, int64_t ldx, double* Y, int64_t ldy, double alpha = 1.0, double beta = 0.0) {
        rep->n_spmm++;
        ab(spmm_b(beta != 0.0));
        tb();
        const int r = spmm_dev(ctx, A, k, X, ldx, nullptr, k, alpha, beta, Y, ldy);
        te(BK_K_SPMM);
        return r;
    }
    int gram(const double* X, int64_t ldx, int ka, const double* Y, int64_t ldy, double* G) {
        rep->n_gram++;
        ab(8 * n * (X == Y && ka == k ? ka : ka + k));
        if (allred) rep->n_allreduce++;
        tb();
        const int r = gram_dev(ctx, n, ka, k, X, ldx, Y, ldy, G, allred);
        te(BK_K_GRAM);
        return r;
    }
    int coldot(const double* X, int64_t ldx, const double* Y, int64_t ldy, const double* Y2, int64_t ldy2,
               double* d, double* d2) {
        tb();
        const int r = coldot_(X, ldx, Y, ldy, Y2, ldy2, d, d2);
        te(BK_K_GRAM);
        return r;
    }
    int coldot_(const double* X, int64_t ldx, const double* Y, int64_t ldy, const double* Y2, int64_t ldy2,
                double* d, double* d2) {
        rep->n_gram++;
        ab(vb() * (1 + (Y != X) + (Y2 != nullptr && Y2 != X && Y2 != Y)));
        double* part = (double*)ws_get(ctx, WS_COLDOT_PART, coldot_ws_doubles(n, k, ctx->num_sms) * sizeof(double));
        double* spart = use_stream_kernels()
                            ? (double*)ws_get(ctx, WS_COLDOT_PART + 32, stream_part_doubles(ctx->num_sms) * sizeof(double))
                            : nullptr;
        if (n > 0 && spart &&
            launch_coldot_stream(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, spart, ctx->d_tickets + 32, ctx->num_sms, st)) {
            // TMA-staged column dots
        } else if (n > 0) {
            launch_coldot(n, k, X, ldx, Y, ldy, Y2, ldy2, d, d2, part, ctx->num_sms, st);
        } else {
            cudaMemsetAsync(d, 0, sizeof(double) * k, st);
            if (d2) cudaMemsetAsync(d2, 0, sizeof(double) * k, st);
        }
        int r = launched("coldot");
        if (r) return r;
        std::vector<std::pair<double*, int64_t>> outs{{d, k}};
        if (d2) outs.push_back({d2, k});
        return reduce_outputs(outs);
    }
    // p > 1: sum a reduction pass's outputs over the ranks -- ONE allreduce when they are adjacent
    // in memory (the solvers lay them out that way), else one per output
    int reduce_outputs(std::vector<std::pair<double*, int64_t>> outs) {
        if (!allred || outs.empty()) return BK_OK;
        std::sort(outs.begin(), outs.end());
        bool adjacent = true;
        for (size_t i = 1; i < outs.size(); ++i) adjacent = adjacent && outs[i - 1].first + outs[i - 1].second == outs[i].first;
        if (adjacent) {
            rep->n_allreduce++;
            return allreduce_sum(ctx, outs[0].first, outs.back().first + outs.back().second - outs[0].first);
        }
        for (auto& o : outs) {
            rep->n_allreduce++;
            int r = allreduce_sum(ctx, o.first, o.second);
            if (r) return r;
        }
        return BK_OK;
    }
    // fused multi-operand Gram (k x k blocks of [arrays[xs..]]^T [arrays[ys..]]), summed over ranks
    int gram_multi(int nxa, const int* xs, int nya, const int* ys, int nin, const double* const* arrays,
                   double* const (*blk)[2], int ndot = 0, const int (*dp)[2] = nullptr, double* const* dots = nullptr,
                   const SmallEpi* epi = nullptr, int cls = BK_K_FUSED_GRAM) {
        rep->n_gram++;
        ab(vb() * nin);
        double* spart = (double*)ws_get(ctx, WS_GRAM_PART + 32, stream_part_doubles(ctx->num_sms) * sizeof(double));
        tb();
        if (!launch_gram_multi_stream(n, k, nxa, xs, nya, ys, nin, arrays, blk, spart, ctx->d_tickets,
                                      ctx->num_sms, st, ndot, dp, dots, epi))
            return set_error(ctx, BK_ERR_UNSUPPORTED, "fused gram not applicable");
        te(cls);
        int r = launched("gram_multi");
        if (r) return r;
        std::vector<std::pair<double*, int64_t>> outs;
        for (int i = 0; i < nxa; ++i)
            for (int j = 0; j < nya; ++j)
                if (blk[i][j]) outs.push_back({blk[i][j], (int64_t)k * k});
        for (int q = 0; q < ndot; ++q) outs.push_back({dots[q], k});
        return reduce_outputs(outs);
    }
    // Y = A X with a reduction in the apply's epilogue (spmm_red_dev; false = not applicable,
    // nothing enqueued): red 1 blk0 = e0^T Y, blk1 = e0^T e1; red 2 blk0 = e0^T Y, dots <Y,X>, <Y,Y>
    bool spmm_red(const double* X, double* Y, int red, const double* e0, const double* e1, double* blk0,
                  double* blk1, double* dot0, double* dot1, const SmallEpi* epi, int* err) {
        tb();
        if (!spmm_red_dev(ctx, A, k, X, Y, red, e0, e1, blk0, blk1, dot0, dot1, epi)) return false;
        te(red == 2 ? BK_K_FUSED_APPLY_DOTS : BK_K_FUSED_APPLY);
        rep->n_spmm++;
        rep->n_gram++;
        ab(spmm_b(false) + (red == 1 ? 2 : (red == 2 ? 1 : 0)) * vb());
        *err = launched("fused apply");
        return true;
    }
    // out = a Xin + s P C (+ w W), optionally halted
    int upd(double* out, int64_t ldo, double a, const double* Xin, int64_t ldxin, double s, const double* P,
            int64_t ldp, int kp, const double* C, const double* W = nullptr, int64_t ldw = 0, double w_host = 0.0,
            const double* w_dev = nullptr, bool halted = true) {
        rep->n_update++;
        ab(8 * n * ((P && kp > 0 ? kp : 0) + k + (a != 0.0 && Xin ? k : 0) + (W ? k : 0)));
        UpdArgs u{};
        u.n = n; u.kp = kp; u.k = k;
        u.a = a; u.Xin = Xin; u.ldxin = ldxin;
        u.s = s; u.P = P; u.ldp = ldp; u.C = C;
        u.W = W; u.ldw = ldw; u.w_host = w_host; u.w_dev = w_dev;
        u.out = out; u.ldo = ldo;
        u.halt = halted ? &ds->halt : nullptr;
        tb();
        launch_update(u, st);
        te(BK_K_UPDATE);
        return launched("update");
    }
    int copy(double* dst, int64_t ldd, const double* src, int64_t lds) {
        ab(2 * vb());
        tb();
        const int r = copy_(dst, ldd, src, lds);
        te(BK_K_COPY);
        return r;
    }
    int copy_(double* dst, int64_t ldd, const double* src, int64_t lds) {
        if (n == 0) return BK_OK;
        if (ldd == k && lds == k)   // contiguous: one linear copy (a 2-D copy of k*8-byte rows is far slower)
            return cuda_check(ctx, cudaMemcpyAsync(dst, src, (size_t)n * k * sizeof(double), cudaMemcpyDeviceToDevice, st),
                              "copy");
        return cuda_check(ctx,
                          cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double), k * sizeof(double),
                                            n, cudaMemcpyDeviceToDevice, st),
                          "copy");
    }
    // R = B - A X  (X = 0: R = B)
    int residual(const double* B, int64_t ldb, const double* X, int64_t ldx, double* R, bool x_zero) {
        int r = copy(R, k, B, ldb);
        if (r || x_zero) return r;
        return spmm(X, ldx, R, k, -1.0, 1.0);
    }
};

#define TRY(x) do { int _r = (x); if (_r) return _r; } while (0)

int finish(Solver& S, const double* B, int64_t ldb, const double* X, int64_t ldx, cudaEvent_t e0) {
    bk_ctx* ctx = S.ctx;
    TRY(S.poll());
    const DevStatus h = *S.hs;
    bk_solve_report* rep = S.rep;
    rep->iterations = h.iter;
    rep->converged = h.converged;
    rep->breakdown_column = h.breakdown_col;
    for (int c = 0; c < S.k; ++c) rep->relres[c] = h.relres[c];
    // true residual, recomputed from scratch (diagnostic)
    double* R = S.vec();
    double* d = S.small(64);
    TRY(S.residual(B, ldb, X, ldx, R, false));
    TRY(S.coldot(R, S.k, R, S.k, nullptr, 0, d, nullptr));
    double* hd = (double*)((char*)ctx->h_pinned + 8192);
    TRY(cuda_check(ctx, cudaMemcpyAsync(hd, d, sizeof(double) * S.k, cudaMemcpyDeviceToHost, S.st), "true res"));
    cudaEvent_t e1;
    cudaEventCreate(&e1);
    cudaEventRecord(e1, S.st);
    TRY(cuda_check(ctx, cudaStreamSynchronize(S.st), "finish"));
    S.tsum();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e1);
    rep->t_total_ms = ms;
    for (int c = 0; c < S.k; ++c) {
        const double r0 = h.r0[c];
        rep->true_relres[c] = std::sqrt(std::max(hd[c], 0.0)) / (r0 > 0.0 ? r0 : 1.0);
    }
    if (h.breakdown_col >= 0) rep->status = BK_BREAKDOWN;
    else if (h.converged) rep->status = BK_OK;
    else rep->status = BK_NOT_CONVERGED;
    return rep->status;
}

// ---------------------------------------------------------------- O4 block CG
// BK_FUSED=0 selects the unfused kernel sequences (A/B comparisons, tests)
static bool fused_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("BK_FUSED");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

int block_cg(Solver& S, const double* B, int64_t ldb, double* X, int64_t ldx, cudaEvent_t e0) {
    const int k = S.k;
    const bool jac = S.o->precond != BK_PRECOND_NONE;   // Jacobi or Chebyshev: Z = M^-1 R
    double* R = S.vec();
    double* P = S.vec();
    double* Q = S.vec();
    double* Z = jac ? S.vec() : R;
    double* sm = S.small(8 * 32 * 32);
    double *PQ = sm, *RZ = sm + 1024, *RZn = sm + 2048, *al = sm + 3072, *be = sm + 4096, *nr = sm + 5120;
    // X0 = 0, no preconditioner, packed aligned B: R0 = P0 = B, read in place by the first
    // iteration (Rin / Pin) -- no setup copies
    const bool b_as_r0 = !jac && S.o->x0_is_zero && ldb == k && ((uintptr_t)B % 16) == 0;
    const double* Rin = R;
    const double* Pin = P;
    if (b_as_r0) {
        Rin = Pin = B;
    } else {
        TRY(S.residual(B, ldb, X, ldx, R, S.o->x0_is_zero));
        if (jac) TRY(S.prec(R, Z));
        TRY(S.copy(P, k, Z, k));
    }
    TRY(S.gram(Rin, k, k, jac ? Z : Rin, k, RZ));
    if (jac) {
        TRY(S.coldot(R, k, R, k, nullptr, 0, nr, nullptr));
        sd_conv_check(nr, 1, k, S.o->rtol, S.o->conv_mode, 1, S.ds, S.st);
    } else {
        sd_conv_check(RZ, k + 1, k, S.o->rtol, S.o->conv_mode, 1, S.ds, S.st);
    }
    const double tol = S.o->breakdown_tol;
    // fused pass structure: Q = A P ; PQ = P^T Q (al solve in its epilogue) ;
    // X += P al, R -= Q al, RZn = R^T R in one pass (test, be solve, RZ roll-over in its
    // epilogue) ; P = R + P be.  13 N x k passes per iteration instead of 14, 4 launches instead of 9.
    const bool fused = !jac && fused_enabled() && use_stream_kernels() && S.n > 0 && k % 4 == 0 && k <= 16 &&
                       ldx == k && ((uintptr_t)X % 16) == 0;
    // (BK_EPI=0: separate one-warp kernels instead of the epilogues -- A/B timing)
    static const int epi_env = env_int("BK_EPI", 1);
    const bool epi = fused && !S.allred && epi_env != 0;
    static const int fa_env = env_int("BK_FUSED_APPLY", 1);
    const bool fapply = epi && fa_env != 0;   // 2-D band plans: P^T Q in the Q = A P apply
    SmallEpi e_al, e_be;
    e_al.kind = 4; e_al.k = k; e_al.st = S.ds; e_al.G = PQ; e_al.Rhs = RZ; e_al.Out = al; e_al.tol = tol;
    e_be.kind = 5; e_be.k = k; e_be.st = S.ds; e_be.g = RZn; e_be.Rhs = RZ; e_be.Out = be; e_be.tol = tol;
    e_be.rtol = S.o->rtol; e_be.conv_mode = S.o->conv_mode;
    auto cg_fused = [&]() -> int {
        int ferr = 0;
        if (fapply && S.spmm_red(Pin, Q, 3, nullptr, nullptr, PQ, nullptr, nullptr, nullptr, &e_al, &ferr)) {
            TRY(ferr);   // P^T Q in the epilogue of the apply that produces Q
        } else {
            TRY(S.spmm(Pin, k, Q, k));
            const double* arr[2] = {Pin, Q};
            const int xs[1] = {0}, ys[1] = {1};
            double* const blk[3][2] = {{PQ, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
            TRY(S.gram_multi(1, xs, 1, ys, 2, arr, blk, 0, nullptr, nullptr, epi ? &e_al : nullptr));
            if (!epi) sd_chol_solve(PQ, RZ, al, k, k, tol, S.ds, S.st);
        }
        S.rep->n_update += 2;
        S.rep->n_gram++;   // the tail's R^T R
        double* spart = (double*)ws_get(S.ctx, WS_GRAM_PART + 32, stream_part_doubles(S.ctx->num_sms) * sizeof(double));
        S.ab(6 * S.vb());   // X, P, R, Q read; X, R written
        S.tb();
        if (!launch_cg_tail_stream(S.n, k, X, R, Pin, Q, al, RZn, &S.ds->halt, spart, S.ctx->d_tickets,
                                   S.ctx->num_sms, S.st, epi ? &e_be : nullptr, Rin))
            return set_error(S.ctx, BK_ERR_UNSUPPORTED, "fused CG tail not applicable");
        S.te(BK_K_FUSED_TAIL);
        TRY(S.launched("cg_tail"));
        if (!epi) {
            if (S.allred) {
                S.rep->n_allreduce++;
                TRY(allreduce_sum(S.ctx, RZn, (int64_t)k * k));
            }
            sd_conv_check(RZn, k + 1, k, S.o->rtol, S.o->conv_mode, 0, S.ds, S.st);
            sd_chol_solve(RZ, RZn, be, k, k, tol, S.ds, S.st);
            std::swap(RZ, RZn);
        }
        S.rep->n_small += 2;
        TRY(S.upd(P, k, 1.0, R, k, 1.0, Pin, k, k, be));
        Rin = R;
        Pin = P;
        return 0;
    };
    auto cg_plain = [&]() -> int {
        TRY(S.spmm(Pin, k, Q, k));
        TRY(S.gram(Pin, k, k, Q, k, PQ));
        sd_chol_solve(PQ, RZ, al, k, k, tol, S.ds, S.st);
        S.rep->n_small++;
        TRY(S.upd(X, ldx, 1.0, X, ldx, 1.0, Pin, k, k, al));
        TRY(S.upd(R, k, 1.0, Rin, k, -1.0, Q, k, k, al));
        if (jac) {
            TRY(S.coldot(R, k, R, k, nullptr, 0, nr, nullptr));
            sd_conv_check(nr, 1, k, S.o->rtol, S.o->conv_mode, 0, S.ds, S.st);
            TRY(S.prec(R, Z));
            TRY(S.gram(R, k, k, Z, k, RZn));
        } else {
            TRY(S.gram(R, k, k, R, k, RZn));
            sd_conv_check(RZn, k + 1, k, S.o->rtol, S.o->conv_mode, 0, S.ds, S.st);
        }
        sd_chol_solve(RZ, RZn, be, k, k, tol, S.ds, S.st);
        S.rep->n_small += 2;
        TRY(S.upd(P, k, 1.0, Z, k, 1.0, Pin, k, k, be));
        std::swap(RZ, RZn);
        Rin = R;
        Pin = P;
        return 0;
    };
    // (the RZ / RZn swap makes two iterations the period of the launch sequence)
    if (fused) TRY(S.iterate(epi ? 1 : 2, cg_fused));
    else TRY(S.iterate(2, cg_plain));
    return finish(S, B, ldb, X, ldx, e0);
}

// ---------------------------------------------------------------- O11 single-reduction block CG
// NEXT-2 (R32): every k x k quantity of an iteration comes from ONE reduction
// pass over [R, W = A R]; Q = A P is carried by a recurrence.  Fused pass structure:
//   tail:  P = R + P be ; Q = W + Q be ; X += P al ; R -= Q al     (one pass, 9 N x k)
//   W = A R with [R^T W, R^T R] in the apply's epilogue (RED 4, X = R from the staged window)
//          -> k x k epilogue: test on diag(R^T R), be, S = R^T W - be^T S be, al
// The first tail runs with P = Q = 0 and be = 0 (P = R, Q = W).  p > 1: the two k x k blocks
// are adjacent, so the pass costs ONE allreduce.
int block_cg1(Solver& S, const double* B, int64_t ldb, double* X, int64_t ldx, cudaEvent_t e0) {
    const int k = S.k;
    double* R = S.vec();
    double* W = S.vec();
    double* P = S.vec();
    double* Q = S.vec();
    double* sm = S.small(8 * 32 * 32);
    double *D = sm, *Gn = sm + k * k, *Gold = sm + 2048, *Sst = sm + 3072, *al = sm + 4096, *be = sm + 5120;
    // X0 = 0 with a packed aligned B: R0 = B, read in place by the setup reduction and the first
    // tail (Rin) -- no copy
    const bool b_as_r0 = S.o->x0_is_zero && ldb == k && ((uintptr_t)B % 16) == 0;
    const double* Rin = R;
    if (b_as_r0) Rin = B;
    else TRY(S.residual(B, ldb, X, ldx, R, S.o->x0_is_zero));
    if (S.n > 0) {
        S.ab(2 * S.vb());
        TRY(cuda_check(S.ctx, cudaMemsetAsync(P, 0, (size_t)S.n * k * sizeof(double), S.st), "P = 0"));
        TRY(cuda_check(S.ctx, cudaMemsetAsync(Q, 0, (size_t)S.n * k * sizeof(double), S.st), "Q = 0"));
    }
    const bool al16 = ((uintptr_t)X % 16) == 0 && ((uintptr_t)R % 16) == 0 && ((uintptr_t)W % 16) == 0 &&
                      ((uintptr_t)Rin % 16) == 0;
    const bool fused = fused_enabled() && use_stream_kernels() && S.n > 0 && k % 4 == 0 && k <= 16 && ldx == k && al16;
    const bool multi = use_stream_kernels() && S.n > 0 && k <= 16 && al16;   // one Gram pass for both blocks
    static const int epi_env = env_int("BK_EPI", 1);
    static const int fa_env = env_int("BK_FUSED_APPLY", 1);
    const bool epi = !S.allred && epi_env != 0;
    SmallEpi e_init, e_it;
    e_it.kind = 6; e_it.k = k; e_it.st = S.ds; e_it.G = D; e_it.g = Gn; e_it.Rhs = Gold; e_it.S = Sst;
    e_it.Out = al; e_it.Out2 = be; e_it.tol = S.o->breakdown_tol; e_it.rtol = S.o->rtol;
    e_it.conv_mode = S.o->conv_mode;
    e_init = e_it;
    e_init.kind = 7;
    // W = A R and the one reduction pass [R^T W, R^T R] (+ its k x k epilogue)
    auto reduce = [&](const SmallEpi& e) -> int {
        int ferr = 0;
        if (epi && fa_env != 0 && S.spmm_red(Rin, W, 4, nullptr, nullptr, D, Gn, nullptr, nullptr, &e, &ferr))
            return ferr;
        TRY(S.spmm(Rin, k, W, k));
        bool ran_epi = false;
        if (multi) {
            const double* arr[2] = {Rin, W};
            const int xs[1] = {0}, ys[2] = {1, 0};
            double* const blk[3][2] = {{D, Gn}, {nullptr, nullptr}, {nullptr, nullptr}};
            TRY(S.gram_multi(1, xs, 2, ys, 2, arr, blk, 0, nullptr, nullptr, epi ? &e : nullptr, BK_K_GRAM));
            ran_epi = epi;
        } else {
            TRY(S.gram(Rin, k, k, W, k, D));
            TRY(S.gram(Rin, k, k, Rin, k, Gn));
        }
        if (!ran_epi) {
            sd_small_epi(e, S.st);
            TRY(S.launched("cg1 step"));
        }
        return 0;
    };
    S.rep->n_small++;
    TRY(reduce(e_init));
    auto body = [&]() -> int {
        S.rep->n_update += 4;
        if (fused) {
            S.ab(9 * S.vb());   // X, R, P, W, Q read; X, R, P, Q written
            S.tb();
            if (!launch_cg1_tail_stream(S.n, k, X, R, P, W, Q, al, be, &S.ds->halt, S.ctx->num_sms, S.st, Rin))
                return set_error(S.ctx, BK_ERR_UNSUPPORTED, "cg1 tail not applicable");
            S.te(BK_K_FUSED_TAIL);
            TRY(S.launched("cg1_tail"));
        } else {
            S.rep->n_update -= 4;   // (upd counts its own)
            TRY(S.upd(P, k, 1.0, Rin, k, 1.0, P, k, k, be));
            TRY(S.upd(Q, k, 1.0, W, k, 1.0, Q, k, k, be));
            TRY(S.upd(X, ldx, 1.0, X, ldx, 1.0, P, k, k, al));
            TRY(S.upd(R, k, 1.0, Rin, k, -1.0, Q, k, k, al));
        }
        S.rep->n_small++;
        Rin = R;
        return reduce(e_it);
    };
    TRY(S.iterate(1, body));
    return finish(S, B, ldb, X, ldx, e0);
}

// ---------------------------------------------------------------- O6 block BiCGStab
// Fused pass structure, same steps and order of the O6 recurrences:
//   V = A P                          (windowed apply)
//   [M1 RR] = Rt^T [V R]             (one pass over Rt, V, R)
//   al = M1^-1 RR ; S = R - V al
//   T = A S
//   RtT = Rt^T T, ts = <T_c,S_c>, tt = <T_c,T_c>   (one pass: DMMA Gram + FMA column dots)
//   w = sum ts / sum tt ; be = -M1^-1 RtT (M1's LU factors from the al solve)
//   X += P al + w S ; R = S - w T ; P = R + (P - w V) be ; rr = ||R_c||^2   (one pass)
//   convergence test on rr
// 21 N x k passes per iteration instead of 28 for the unfused sequence.

int block_bicgstab(Solver& S, const double* B, int64_t ldb, double* X, int64_t ldx, cudaEvent_t e0) {
    const int k = S.k;
    double* R = S.vec();
    double* Rt_buf = S.vec();
    double* P = S.vec();
    double* V = S.vec();
    double* Sv = S.vec();
    double* T = S.vec();
    double* Tmp = S.vec();
    double* sm = S.small(8 * 32 * 32);
    // the outputs of one reduction pass are adjacent ([M1 RR], [RtT ts tt]): with p > 1 each
    // pass is summed by ONE allreduce (Solver::reduce_outputs)
    double *M1 = sm, *RR = sm + k * k, *RtT = sm + 2048, *ts = RtT + k * k, *tt = ts + k, *al = sm + 3200,
           *be = sm + 4224, *nr = sm + 5248, *LUf = sm + 6144;
    int* piv = reinterpret_cast<int*>(sm + 7168);
    // X0 = 0 with a packed, aligned B: R0 = P0 = Rt = B.  Rt is never written, and the first
    // iteration reads B in place of R and P (Rin / Pin), so the setup copies nothing.
    const bool b_as_r0 = S.o->x0_is_zero && ldb == k && ((uintptr_t)B % 16) == 0;
    const double* Rin = R;
    const double* Pin = P;
    const double* Rt = Rt_buf;
    if (b_as_r0) {
        Rin = Pin = Rt = B;
    } else {
        TRY(S.residual(B, ldb, X, ldx, R, S.o->x0_is_zero));
        TRY(S.copy(Rt_buf, k, R, k));
        TRY(S.copy(P, k, R, k));
    }
    TRY(S.coldot(Rin, k, Rin, k, nullptr, 0, nr, nullptr));
    sd_conv_check(nr, 1, k, S.o->rtol, S.o->conv_mode, 1, S.ds, S.st);
    const double tol = S.o->breakdown_tol;
    const double* om = &S.ds->omega;
    const double* nom = &S.ds->neg_omega;
    // (k a multiple of 4: the tail pads its last 8-column block; the column dots ride in the
    // RtT pass only when k divides 32, else they take one coldot pass before it)
    const bool fused = fused_enabled() && use_stream_kernels() && S.n > 0 && k % 4 == 0 && k <= 16 &&
                       ldx == k && ((uintptr_t)X % 16) == 0;
    const bool dots_fused = (32 % k) == 0;
    // one rank: the k x k steps run in the epilogue of the pass that produces their
    // input (no separate small-kernel launches); p > 1: after the allreduce
    // (BK_EPI=0: separate one-warp kernels instead of the epilogues -- A/B timing)
    static const int epi_env = env_int("BK_EPI", 1);
    const bool epi = fused && !S.allred && epi_env != 0;
    SmallEpi e_al, e_be, e_cv;
    e_al.kind = 1; e_al.k = k; e_al.st = S.ds; e_al.G = M1; e_al.Rhs = RR; e_al.Out = al; e_al.sign = 1.0;
    e_al.tol = tol; e_al.LU = LUf; e_al.piv = piv;
    e_be.kind = 2; e_be.k = k; e_be.st = S.ds; e_be.ts = ts; e_be.tt = tt; e_be.Rhs = RtT; e_be.Out = be;
    e_be.sign = -1.0; e_be.LU = LUf; e_be.piv = piv;
    e_cv.kind = 3; e_cv.k = k; e_cv.st = S.ds; e_cv.g = nr; e_cv.rtol = S.o->rtol; e_cv.conv_mode = S.o->conv_mode;
    // one rank, 2-D band plan: the Rt^T [V R] and Rt^T T, <T,S>, <T,T> passes ride in the
    // epilogues of the applies that produce V and T (BK_FUSED_APPLY=0: separate)
    static const int fa_env = env_int("BK_FUSED_APPLY", 1);
    const bool fapply = fused && epi && fa_env != 0;
    auto iteration = [&]() -> int {
        int ferr = 0;
        if (fapply && S.spmm_red(Pin, V, 1, Rt, Rin, M1, RR, nullptr, nullptr, &e_al, &ferr)) {
            TRY(ferr);
            TRY(S.upd(Sv, k, 1.0, Rin, k, -1.0, V, k, k, al));
            if (S.spmm_red(Sv, T, 2, Rt, nullptr, RtT, nullptr, ts, tt, &e_be, &ferr)) {
                TRY(ferr);
            } else {
                TRY(S.spmm(Sv, k, T, k));
                const double* arr[3] = {Rt, Sv, T};
                const int xs[1] = {0}, ys[1] = {2};
                double* const blk[3][2] = {{RtT, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
                const int dp[2][2] = {{2, 1}, {2, 2}};
                double* const dots[2] = {ts, tt};
                if (!dots_fused) TRY(S.coldot(T, k, Sv, k, T, k, ts, tt));
                TRY(S.gram_multi(1, xs, 1, ys, 3, arr, blk, dots_fused ? 2 : 0, dp, dots, &e_be, BK_K_FUSED_DOTS));
            }
            S.rep->n_update += 3;
            double* spart = (double*)ws_get(S.ctx, WS_GRAM_PART + 32, stream_part_doubles(S.ctx->num_sms) * sizeof(double));
            S.ab(8 * S.vb());   // X, P, S, T, V read; X, R, P written
            S.tb();
            if (!launch_bcg_tail_stream(S.n, k, X, R, P, Sv, T, V, al, be, om, nr, &S.ds->halt, spart,
                                        S.ctx->d_tickets, S.ctx->num_sms, S.st, &e_cv, Pin))
                return set_error(S.ctx, BK_ERR_UNSUPPORTED, "fused BiCGStab tail not applicable");
            S.te(BK_K_FUSED_TAIL);
            TRY(S.launched("bcg_tail"));
            S.rep->n_small += 4;
            Rin = R;
            Pin = P;
            return 0;
        }
        TRY(S.spmm(Pin, k, V, k));
        if (fused) {
            const double* arr[3] = {Rt, V, Rin};
            const int xs[1] = {0}, ys[2] = {1, 2};
            double* const blk[3][2] = {{M1, RR}, {nullptr, nullptr}, {nullptr, nullptr}};
            TRY(S.gram_multi(1, xs, 2, ys, 3, arr, blk, 0, nullptr, nullptr, epi ? &e_al : nullptr));
            if (!epi) sd_lu_solve(M1, RR, al, k, k, 1.0, tol, S.ds, S.st, 0, LUf, piv);   // factors kept for be
        } else {
            TRY(S.gram(Rt, k, k, V, k, M1));
            TRY(S.gram(Rt, k, k, Rin, k, RR));
            sd_lu_solve(M1, RR, al, k, k, 1.0, tol, S.ds, S.st);
        }
        TRY(S.upd(Sv, k, 1.0, Rin, k, -1.0, V, k, k, al));
        TRY(S.spmm(Sv, k, T, k));
        if (fused) {
            const double* arr[3] = {Rt, Sv, T};
            const int xs[1] = {0}, ys[1] = {2};
            double* const blk[3][2] = {{RtT, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
            const int dp[2][2] = {{2, 1}, {2, 2}};   // <T,S>, <T,T> per column
            double* const dots[2] = {ts, tt};
            if (!dots_fused) TRY(S.coldot(T, k, Sv, k, T, k, ts, tt));   // before the pass whose epilogue uses them
            TRY(S.gram_multi(1, xs, 1, ys, 3, arr, blk, dots_fused ? 2 : 0, dp, dots, epi ? &e_be : nullptr,
                             BK_K_FUSED_DOTS));
            if (!epi) {
                sd_omega(ts, tt, k, S.ds, S.st);
                sd_lu_resolve(LUf, piv, RtT, be, k, k, -1.0, S.ds, S.st);   // same M1: no new breakdown
            }
            S.rep->n_update += 3;
            S.rep->n_gram++;
            double* spart = (double*)ws_get(S.ctx, WS_GRAM_PART + 32, stream_part_doubles(S.ctx->num_sms) * sizeof(double));
            S.ab(8 * S.vb());   // X, P, S, T, V read; X, R, P written
            S.tb();
            if (!launch_bcg_tail_stream(S.n, k, X, R, P, Sv, T, V, al, be, om, nr, &S.ds->halt, spart,
                                        S.ctx->d_tickets, S.ctx->num_sms, S.st, epi ? &e_cv : nullptr, Pin))
                return set_error(S.ctx, BK_ERR_UNSUPPORTED, "fused BiCGStab tail not applicable");
            S.te(BK_K_FUSED_TAIL);
            TRY(S.launched("bcg_tail"));
            if (S.allred) {
                S.rep->n_allreduce++;
                TRY(allreduce_sum(S.ctx, nr, k));
            }
            if (!epi) sd_conv_check(nr, 1, k, S.o->rtol, S.o->conv_mode, 0, S.ds, S.st);
            S.rep->n_small += 4;
        } else {
            TRY(S.coldot(T, k, Sv, k, T, k, ts, tt));
            sd_omega(ts, tt, k, S.ds, S.st);
            TRY(S.upd(X, ldx, 1.0, X, ldx, 1.0, Pin, k, k, al, Sv, k, 1.0, om));
            TRY(S.upd(R, k, 1.0, Sv, k, 0.0, nullptr, k, 0, nullptr, T, k, 1.0, nom));
            TRY(S.coldot(R, k, R, k, nullptr, 0, nr, nullptr));
            sd_conv_check(nr, 1, k, S.o->rtol, S.o->conv_mode, 0, S.ds, S.st);
            TRY(S.gram(Rt, k, k, T, k, RtT));
            sd_lu_solve(M1, RtT, be, k, k, -1.0, tol, S.ds, S.st);
            S.rep->n_small += 4;
            TRY(S.upd(Tmp, k, 1.0, Pin, k, 0.0, nullptr, k, 0, nullptr, V, k, 1.0, nom));
            TRY(S.upd(P, k, 1.0, R, k, 1.0, Tmp, k, k, be));
        }
        Rin = R;
        Pin = P;
        return 0;
    };
    TRY(S.iterate(1, iteration));
    return finish(S, B, ldb, X, ldx, e0);
}

// ---------------------------------------------------------------- O5 block GMRES(m)
int block_gmres(Solver& S, const double* B, int64_t ldb, double* X, int64_t ldx, cudaEvent_t e0) {
    const int k = S.k, m = S.o->restart;
    // basis: one row-major n x (m+1)k array, V_j = columns [jk, (j+1)k)
    const int64_t ldv = (int64_t)(m + 1) * k;
    double* Vb = S.vec((int)((m + 1) * k));
    auto Vblk = [&](int j) { return Vb + (int64_t)j * k; };
    double* W = S.vec();
    const size_t hk = (size_t)(m + 1) * k * k;
    double* Hcol = S.small(hk);
    double* H1 = S.small(hk);
    double* H2 = S.small(hk);
    double* g = S.small(hk);
    double* Qs = S.small((size_t)m * 4 * k * k);
    const int ldr = m * k;
    double* Rtri = S.small((size_t)ldr * ldr);
    double* y = S.small((size_t)m * k * k);
    double* sm = S.small(8 * 32 * 32);
    double *G1 = sm, *R1 = sm + 1024, *R1i = sm + 2048, *R2i = sm + 3072, *Sr = sm + 4096, *nr = sm + 5120;
    // CholQR2 (O5): Q1 = W R1^-1 with R1^T R1 = W^T W; R2^T R2 = Q1^T Q1; V = Q1 R2^-1, R = R2 R1.
    // Q1 goes to a contiguous scratch (streaming Gram, no strided read-back) and the basis
    // block is written once from W with the product R1^-1 R2^-1 (no in-place strided pass).
    double* Q1 = S.vec();
    double* R12i = S.small(32 * 32);
    const double tol = S.o->breakdown_tol;
    // (small systems are launch-bound: there the two-pass in-place form with one launch fewer)
    const bool small_n = S.n < 65536;
    // [V_0 .. V_{nb-1}]^T Wm -> Hout (nb k x k): one strided multi-Gram
    auto gram_basis = [&](int nb, const double* Wm, double* Hout) -> int {
        return S.gram(Vb, ldv, nb * k, Wm, k, Hout);
    };
    // out = a Xin + s [V_0 .. V_{nb-1}] Hc (nb k x k): one strided multi-update
    auto upd_basis = [&](double* out, int64_t ldo, double a, const double* Xin, double s, int nb, const double* Hc,
                         bool halted) -> int {
        return S.upd(out, ldo, a, Xin, ldo, s, Vb, ldv, nb * k, Hc, nullptr, 0, 0.0, nullptr, halted);
    };
    auto cholqr2 = [&](const double* Wm, double* Vout, double* Rprod) -> int {
        TRY(S.gram(Wm, k, k, Wm, k, G1));
        sd_chol_qr(G1, R1, R1i, nullptr, nullptr, k, tol, S.ds, S.st);
        if (small_n) {
            TRY(S.upd(Vout, ldv, 0.0, nullptr, 0, 1.0, Wm, k, k, R1i));
            TRY(S.gram(Vout, ldv, k, Vout, ldv, G1));
            sd_chol_qr(G1, nullptr, R2i, R1, Rprod, k, tol, S.ds, S.st);
            return S.upd(Vout, ldv, 0.0, nullptr, 0, 1.0, Vout, ldv, k, R2i);
        }
        TRY(S.upd(Q1, k, 0.0, nullptr, 0, 1.0, Wm, k, k, R1i));
        TRY(S.gram(Q1, k, k, Q1, k, G1));
        sd_chol_qr(G1, nullptr, R2i, R1, Rprod, k, tol, S.ds, S.st);
        {   // R12i = R1^-1 R2^-1 (k x k, an update over k rows)
            UpdArgs u{};
            u.n = k; u.kp = k; u.k = k; u.a = 0.0; u.s = 1.0; u.P = R1i; u.ldp = k; u.C = R2i;
            u.out = R12i; u.ldo = k; u.halt = &S.ds->halt;
            launch_update(u, S.st);
            TRY(S.launched("cholqr2 R12i"));
        }
        return S.upd(Vout, ldv, 0.0, nullptr, 0, 1.0, Wm, k, k, R12i);
    };
    TRY(S.residual(B, ldb, X, ldx, W, S.o->x0_is_zero));
    TRY(S.coldot(W, k, W, k, nullptr, 0, nr, nullptr));
    sd_conv_check(nr, 1, k, S.o->rtol, S.o->conv_mode, 1, S.ds, S.st);
    int it = 0;
    bool done = false;
    while (!done && it < S.o->max_iters) {
        cudaMemsetAsync(&S.ds->gm_steps, 0, sizeof(int), S.st);
        cudaMemsetAsync(g, 0, hk * sizeof(double), S.st);
        cudaMemsetAsync(Rtri, 0, (size_t)ldr * ldr * sizeof(double), S.st);
        // [V_0, S] = CholQR2(R)
        TRY(cholqr2(W, Vblk(0), Sr));
        sd_copy(Sr, g, k * k, S.st);
        int j = 0;
        for (; j < m; ++j) {
            double* Vj = Vblk(j);
            double* Vn = Vblk(j + 1);
            const int ka = (j + 1) * k;
            TRY(S.spmm(Vj, ldv, W, k));
            // BCGS2: two passes of Hp = V^T W; W -= V Hp
            TRY(gram_basis(j + 1, W, H1));
            TRY(upd_basis(W, k, 1.0, W, -1.0, j + 1, H1, true));
            TRY(gram_basis(j + 1, W, H2));
            TRY(upd_basis(W, k, 1.0, W, -1.0, j + 1, H2, true));
            sd_add(H1, H2, Hcol, ka * k, S.st);
            // [V_{j+1}, H_{j+1,j}] = CholQR2(W)
            TRY(cholqr2(W, Vn, Hcol + (int64_t)ka * k));
            sd_gmres_step(Hcol, j, k, Qs, Rtri, ldr, g, S.o->rtol, S.o->conv_mode, S.ds, S.st);
            S.rep->n_small += 5;
            ++it;
            if (it % S.o->check_every == 0 || it >= S.o->max_iters || j + 1 == m) {
                TRY(S.poll());
                if (S.hs->halt) { done = true; break; }
            }
            if (it >= S.o->max_iters) { done = true; break; }
        }
        // X += [V_0 .. V_{s-1}] y,  R y = g  (s completed steps of this cycle)
        TRY(S.poll());
        const int steps = S.hs->gm_steps;
        if (S.hs->halt) done = true;
        if (steps > 0) {
            sd_gmres_backsolve(Rtri, ldr, g, y, steps * k, k, S.st);
            TRY(upd_basis(X, ldx, 1.0, X, 1.0, steps, y, false));
        }
        if (!done && it < S.o->max_iters) TRY(S.residual(B, ldb, X, ldx, W, false));
    }
    return finish(S, B, ldb, X, ldx, e0);
}

}  // namespace

int solve_impl(bk_ctx* ctx, const bk_csr* A, int k, const double* B, int64_t ldb, double* X, int64_t ldx,
               const bk_solve_opts* o, bk_solve_report* rep) {
    memset(rep, 0, sizeof *rep);
    rep->breakdown_column = -1;
    Solver S{ctx, A, A->n_local, k, o, rep, ctx->stream};
    S.allred = ctx->nranks > 1;
    cudaEvent_t e0;
    cudaEventCreate(&e0);
    cudaEventRecord(e0, S.st);
    int r = S.init_status();
    if (!r && o->x0_is_zero && A->n_local > 0)
        r = cuda_check(ctx,
                       ldx == k ? cudaMemsetAsync(X, 0, (size_t)A->n_local * k * sizeof(double), S.st)
                                : cudaMemset2DAsync(X, ldx * sizeof(double), 0, k * sizeof(double), A->n_local, S.st),
                       "zero X");
    if (!r) {
        switch (o->method) {
            case BK_CG: r = block_cg(S, B, ldb, X, ldx, e0); break;
            case BK_GMRES: r = block_gmres(S, B, ldb, X, ldx, e0); break;
            case BK_CG1: r = block_cg1(S, B, ldb, X, ldx, e0); break;
            default: r = block_bicgstab(S, B, ldb, X, ldx, e0); break;
        }
    }
    cudaEventDestroy(e0);
    return r;
}

}  // namespace bk
