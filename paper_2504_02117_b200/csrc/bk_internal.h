// bk_internal.h -- private declarations of the B200 (sm_100a) block-Krylov library.
// Nothing here is shared with oracle/ (the CPU checker); see DESIGN.md §1.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "bk.h"

#ifndef BK_NO_NCCL
#include <nccl.h>
#endif

#include <atomic>

namespace bk {

struct LocalHub;   // in-process loopback transport (comm.cpp)

// Every kernel launch of the library goes through BK_KERNEL so the process-wide
// count is exact (bk_kernel_launch_count(); bench.py reports it as gpu_launches).
extern std::atomic<long long> g_launches;
#define BK_KERNEL(...) (++::bk::g_launches, __VA_ARGS__)

// ------------------------------------------------------------------ device status
// Written by the small-dense / convergence kernels, polled by the host driver.
// `halt` makes every later update kernel of the solve a no-op, so X keeps the
// last good iterate whatever the host polling period is.
struct DevStatus {
    int halt;            // 1 after convergence or breakdown
    int converged;
    int breakdown_col;   // -1 if none
    int iter;            // completed (un-halted) iterations
    int gm_steps;        // GMRES: completed inner steps in the current cycle
    int pending_bd;      // deferred breakdown (column + 1) of an LU solve whose
                         // result is only needed if the next convergence test fails
    int pad[2];
    double relres[BK_MAX_K];
    double r0[BK_MAX_K];
    double omega;        // BiCGStab scalar
    double neg_omega;
};

// ------------------------------------------------------------------ kernel args
struct SpmmArgs {
    const int32_t* rp;      // row pointers (local rows)
    const int32_t* col;     // local column ids (ghost ids >= ncol_local)
    const double* val;
    const int32_t* rows;    // optional explicit row list (boundary rows); null = contiguous
    int64_t row0;           // first row (contiguous mode)
    int64_t nrows;
    const double* X;
    int64_t ldx;
    const double* Xg;       // ghost rows (ld = ldg), column c >= ncol_local -> Xg[c - ncol_local]
    int64_t ldg;
    int32_t ncol_local;
    const double* C;        // k x kout row-major, or null (identity)
    int k, kout;
    double alpha, beta;
    double* Y;
    int64_t ldy;
    // pipe kernel, 3-D lattices: y-slab tile order (sl_S > 0): slab s of sl_L lines, then z,
    // then the line, then the x block (sl_tpl tiles per line) -- keeps the z-neighbour planes
    // of the rows in flight L2-resident when whole planes do not fit
    int sl_S, sl_L, sl_tpl, sl_ny, sl_nz;
    // persistent grids: SMs to size the grid for (0 = all).  p > 1: the interior apply leaves
    // SMs free for NCCL's send/recv kernels while the halo is in flight (abi.cpp)
    int grid_sms;
};

// out = a*Xin + s*(P C) + (w_host * (*w_dev)) * W     (any term may be absent)
struct UpdArgs {
    int64_t n;
    int kp, k;
    double a;
    const double* Xin; int64_t ldxin;
    double s;
    const double* P; int64_t ldp;
    const double* C;        // kp x k row-major (device)
    double w_host;
    const double* w_dev;    // optional device scalar multiplying w_host
    const double* W; int64_t ldw;
    double* out; int64_t ldo;
    const int* halt;        // optional: skip when *halt != 0
};

void launch_bspmm(const SpmmArgs& a, cudaStream_t st);
// Windowed apply (X rows of each diagonal band staged in shared memory by
// TMA) over the planned contiguous row range; false = not
// applicable (the caller then uses launch_bspmm).
struct BandPlan {
    int nbands = 0, extra = 0, max_row_nnz = 0;
    int lo[BK_BAND_MAX] = {}, hi[BK_BAND_MAX] = {};
    int dmin[BK_BAND_MAX] = {}, dmax[BK_BAND_MAX] = {};
    int64_t row0 = 0, nrows = 0;     // planned contiguous row range
};
bool launch_bspmm_win(const SpmmArgs& a, const BandPlan& b, cudaStream_t st);
// The windowed apply with a fused reduction epilogue (the fused block-BiCGStab passes,
// DESIGN.md §4.4; 2-D band plans, k = 8 / 12 / 16, alpha 1, beta 0); false = not applicable:
//   red 1: ro.blk[0][0] = e0^T Y, ro.blk[0][1] = e0^T e1
//   red 2: ro.blk[0][0] = e0^T Y, ro.dots[0] = <Y_c, X_c>, ro.dots[1] = <Y_c, Y_c>
//   red 3: ro.blk[0][0] = X^T Y (no extra operand)
// reduced over the grid in a fixed order; the final CTA runs the k x k epilogue epi (may be null).
struct RedOut;
struct SmallEpi;
bool launch_bspmm_win_red(const SpmmArgs& a, const BandPlan& b, cudaStream_t st, int red, const double* e0,
                          const double* e1, const RedOut& ro, const SmallEpi* epi);
void launch_update(const UpdArgs& a, cudaStream_t st);
// G (ka x kb, row-major, device) = X^T Y; `partials` workspace of gram_ws_doubles().
size_t gram_ws_doubles(int64_t n, int ka, int kb, int num_sms);
void launch_gram(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y,
                 int64_t ldy, double* G, double* partials, int num_sms, cudaStream_t st);
// Same on the FP64 tensor cores (DMMA m8n8k4), one launch; `ticket` is a zeroed
// device int (the last CTA reduces and resets it).
size_t gram_mma_ws_doubles(int64_t n, int ka, int kb, int num_sms);
void launch_gram_mma(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                     double* G, double* part, int* ticket, int num_sms, cudaStream_t st);
// TMA-staged streaming versions (stream.cu); return false when not applicable
// (strided / > 32-wide operands), the caller then uses the generic kernels.
size_t stream_part_doubles(int num_sms);
bool launch_update_stream(const UpdArgs& u, int num_sms, cudaStream_t st);
bool launch_gram_stream(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                        double* G, double* part, int* ticket, int num_sms, cudaStream_t st);
bool launch_coldot_stream(int64_t n, int k, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                          const double* Y2, int64_t ldy2, double* d, double* d2, double* part, int* ticket,
                          int num_sms, cudaStream_t st);
bool use_stream_kernels();
// k <= 4 Gram / update without the TMA ring (flat.cu); false = not applicable
size_t flat_part_doubles(int num_sms);
bool launch_gram_flat(int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                      double* G, double* part, int* ticket, int num_sms, cudaStream_t st);
bool launch_update_flat(const UpdArgs& u, int num_sms, cudaStream_t st);
// Wide / strided multi-Gram and multi-update (wide.cu; GMRES basis, ld = (m+1)k).
size_t gram_wide_ws_doubles(int ka, int kb, int num_sms);
bool launch_gram_wide(int64_t n, int ka, int kb, const double* V, int64_t ldv, const double* W, int64_t ldw,
                      double* G, double* part, int num_sms, cudaStream_t st);
bool launch_update_wide(const UpdArgs& u, cudaStream_t st);
// k x k epilogue of a fused reduction pass, run by the CTA that produced the
// final result (dense_dev.cuh run_small_epi): 1 Out = G^{-1}(sign Rhs) by LU,
// factors kept in LU/piv; 2 BiCGStab omega from ts, tt then Out = G^{-1}(sign Rhs)
// from LU/piv; 3 convergence test on column norms g; 4 Out = G^{-1} Rhs by
// Cholesky (block CG alpha); 5 block CG: convergence test on diag(g), then
// Out = Rhs^{-1} g by Cholesky (beta) and Rhs <- g; 6 / 7 single-reduction block CG step /
// setup (O11; dense_dev.cuh): S state, Out = alpha, Out2 = beta.
struct SmallEpi {
    int kind = 0;
    int k = 0;
    DevStatus* st = nullptr;
    const double* G = nullptr;
    const double* Rhs = nullptr;
    double* Out = nullptr;
    double sign = 1.0, tol = 0.0;
    double* LU = nullptr;
    int* piv = nullptr;
    const double* ts = nullptr;
    const double* tt = nullptr;
    const double* g = nullptr;
    double rtol = 0.0;
    int conv_mode = 0;
    double* S = nullptr;
    double* Out2 = nullptr;
};
// run a SmallEpi as a one-warp kernel (no fused reduction pass: p > 1, or not applicable)
void sd_small_epi(const SmallEpi& e, cudaStream_t s);
// Fused block-BiCGStab passes (stream.cu; false = not applicable):
// multi-operand Gram: X = [arrays[xs[0]] ..], Y = [arrays[ys[0]] ..], all kw wide
// (kw <= 16); k x k block (i, j) of X^T Y is written to blk[i][j] (null = dropped).
// ndot (<= 2) column dots dots[q][c] = sum_r A_q[r,c] B_q[r,c], A_q = arrays[dpair[q][0]],
// B_q = arrays[dpair[q][1]] (kw | 32), computed in the same pass.
bool launch_gram_multi_stream(int64_t n, int kw, int nxa, const int* xs, int nya, const int* ys, int nin,
                              const double* const* arrays, double* const (*blk)[2], double* part, int* ticket,
                              int num_sms, cudaStream_t st, int ndot = 0, const int (*dpair)[2] = nullptr,
                              double* const* dots = nullptr, const SmallEpi* epi = nullptr);
// block CG tail: X += P al; R -= Q al; G = R^T R (new R); k % 8 == 0
// (Rin: where the old R is read, default R -- the first iteration reads R0 = B in place)
bool launch_cg_tail_stream(int64_t n, int k, double* X, double* R, const double* P, const double* Q,
                           const double* al, double* G, const int* halt, double* part, int* ticket, int num_sms,
                           cudaStream_t st, const SmallEpi* epi = nullptr, const double* Rin = nullptr);
// single-reduction block CG tail (O11): P = R + P be; Q = W + Q be; X += P al; R -= Q al
// (new P, Q); k % 4 == 0, k <= 16
bool launch_cg1_tail_stream(int64_t n, int k, double* X, double* R, double* P, const double* W, double* Q,
                            const double* al, const double* be, const int* halt, int num_sms, cudaStream_t st,
                            const double* Rin = nullptr);
// X += P al + w S; R = S - w T; P = R + (P - w V) be; rr_c = ||R_c||^2 (w = *w_dev); k % 8 == 0
// (Pin: where the old P is read, default P)
bool launch_bcg_tail_stream(int64_t n, int k, double* X, double* R, double* P, const double* S, const double* T,
                            const double* V, const double* al, const double* be, const double* w_dev, double* rr,
                            const int* halt, double* part, int* ticket, int num_sms, cudaStream_t st,
                            const SmallEpi* epi = nullptr, const double* Pin = nullptr);
// d[c] = sum_i X[i,c] Y[i,c] for c < k (and optionally d2 with Y2); deterministic.
size_t coldot_ws_doubles(int64_t n, int k, int num_sms);
void launch_coldot(int64_t n, int k, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                   const double* Y2, int64_t ldy2, double* d, double* d2, double* partials,
                   int num_sms, cudaStream_t st);
void launch_row_scale(int64_t n, int k, const double* dinv, const double* X, int64_t ldx,
                      double* out, int64_t ldo, cudaStream_t st);
// NEXT-4 Chebyshev preconditioner (solve.cpp cheb_apply; oracle O9)
void launch_cheb_step(int64_t n, int k, const double* R, int64_t ldr, const double* AZ, const double* dinv,
                      double* W, double* Z, int64_t ldz, double cw, double cr, cudaStream_t st);
void launch_gershgorin(int64_t n, const int32_t* rp, const double* val, const double* dinv, unsigned long long* out,
                       cudaStream_t st);
int allreduce_max(bk_ctx* ctx, double* d, int64_t n);
int alg1_impl(bk_ctx* ctx, const bk_dr_problem* pb, int m, const double* A, int n_steps, int w, double eps,
              int max_newton, const bk_solve_opts* inner, double* traj, int64_t ldt, int* newton_its,
              bk_alg1_report* rep);
// NEXT-3 nonlinear diffusion-reaction operator (nonlin.cu; oracle O10)
void launch_dr_f(int64_t nx, int64_t ny, int64_t nz, double h, const double* Y, int64_t ldy, int w,
                 const double* sinT, const double* g, double* F, int64_t ldf, cudaStream_t st);
void launch_dr_jac(int64_t nx, int64_t ny, int64_t nz, double h, const double* u, int64_t ldu, double shift,
                   double scale, const int32_t* rp, const int32_t* col, double* val, int* bad, cudaStream_t st);
int env_int(const char* name, int dflt);   // integer environment knob (A/B experiments)
// Chebyshev interval after defaults (lmax <= 0: Gershgorin, lmin <= 0: lmax / 30)
void cheb_bounds(const bk_csr* A, const bk_solve_opts* o, double* lmin, double* lmax);
bool cheb_opts_ok(const bk_csr* A, const bk_solve_opts* o);
// Z = M^-1 R (solve.cpp); collective for nranks > 1
int precond_apply_impl(bk_ctx* ctx, const bk_csr* A, int k, const bk_solve_opts* o, const double* R, int64_t ldr,
                       double* Z, int64_t ldz);
void launch_extract_diag_inv(int64_t n, int64_t row_offset, const int32_t* rp, const int32_t* col,
                             const double* val, double* dinv, cudaStream_t st);
void launch_fill(double* p, int64_t n, double v, cudaStream_t st);
void launch_pack_rows(int64_t nrows, int k, const int32_t* rows, const double* X, int64_t ldx,
                      double* out, cudaStream_t st);

// ------------------------------------------------------------------ small dense (1 CTA)
// Out(k x nrhs) = G^{-1} Rhs by Cholesky; breakdown -> st->breakdown_col, st->halt.
void sd_chol_solve(const double* G, const double* Rhs, double* Out, int k, int nrhs, double tol,
                   DevStatus* st, cudaStream_t s);
// Out = G^{-1} (sign * Rhs) by LU with partial pivoting.  defer: a breakdown
// only records st->pending_bd (acted on by the next sd_conv_check if that test
// does not converge) instead of halting.
// LUo / pivo (optional, k x k and k ints): keep the factors for sd_lu_resolve.
void sd_lu_solve(const double* G, const double* Rhs, double* Out, int k, int nrhs, double sign,
                 double tol, DevStatus* st, cudaStream_t s, int defer = 0, double* LUo = nullptr,
                 int* pivo = nullptr);
// Out = G^{-1} (sign Rhs) reusing sd_lu_solve's factors of G (no breakdown possible).
void sd_lu_resolve(const double* LU, const int* piv, const double* Rhs, double* Out, int k, int nrhs, double sign,
                   DevStatus* st, cudaStream_t s);
// R upper (G = R^T R) and Rinv; also Racc <- R * Racc_in if Racc_in != null (Racc = R2 R1).
void sd_chol_qr(const double* G, double* R, double* Rinv, const double* Rprev, double* Rprod,
                int k, double tol, DevStatus* st, cudaStream_t s);
// Convergence test: rel_c = sqrt(max(g_c,0)) / r0_c; sets converged/halt, iter++.
// init != 0: store r0_c = sqrt(g_c) instead.
void sd_conv_check(const double* g, int gstride, int k, double rtol, int conv_mode, int init,
                   DevStatus* st, cudaStream_t s);
// BiCGStab omega = sum(ts) / sum(tt) into st->omega (breakdown if tt == 0);
// ts[c * stride], tt[c * stride] (stride k + 1: diagonals of k x k Grams).
void sd_omega(const double* ts, const double* tt, int k, DevStatus* st, cudaStream_t s, int stride = 1);
// Copy a k x k matrix (device) (used to roll RZ <- RZn).
void sd_copy(const double* src, double* dst, int n, cudaStream_t s);
// GMRES: apply stored rotations Q_0..Q_{j-1} to the new block column, QR the
// 2k x k bottom block into Q_j, rotate g, write residual norms and test.
void sd_gmres_step(double* Hcol, int j, int k, double* Qs, double* Rtri, int ldr, double* g,
                   double rtol, int conv_mode, DevStatus* st, cudaStream_t s);
// GMRES: solve Rtri[0:nk,0:nk] y = g[0:nk] (upper triangular), y: nk x k.
void sd_gmres_backsolve(const double* Rtri, int ldr, const double* g, double* y, int nk, int k,
                        cudaStream_t s);
// H column assembly: Hc = H1 + H2 (n doubles)
void sd_add(const double* a, const double* b, double* out, int n, cudaStream_t s);

}  // namespace bk

// ------------------------------------------------------------------ context / matrix
struct bk_buf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct bk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    int num_sms = 148;
    int sticky = 0;
    std::string last_error;
    cudaStream_t cap_stream = nullptr;   // CUDA graph capture (bk_solve_opts.use_graphs)
    std::vector<bk_buf> ws;       // slot-indexed grow-only device workspaces
    double* h_pinned = nullptr;   // pinned host staging for small results
    int* d_tickets = nullptr;     // zeroed device counters for last-CTA reductions
    size_t h_pinned_bytes = 0;
    int nranks = 1, rank = 0;
    std::vector<bk_csr*> mats;    // live matrices (detached when the ctx is destroyed)
    std::vector<cudaEvent_t> tev; // event pool of the solver's per-kernel timing (opts.timing)
#ifndef BK_NO_NCCL
    ncclComm_t comm = nullptr;
#endif
    bk::LocalHub* hub = nullptr;  // loopback transport instead of NCCL (bk_ctx_set_comm_local)
};

struct bk_neighbor {
    int rank = -1;
    int64_t recv_off = 0, recv_cnt = 0;   // rows into the ghost buffer
    int64_t send_cnt = 0;
    int32_t* d_send_rows = nullptr;       // local row ids to send
    int send_contig = 0;
    int64_t send_begin = 0;
    int64_t send_off = 0;                 // offset (rows) in the packed send buffer
};

struct bk_csr {
    bk_ctx* ctx = nullptr;
    int64_t n_global = 0, row_begin = 0, n_local = 0, nnz = 0;
    int32_t* d_rp = nullptr;
    int32_t* d_col = nullptr;             // local numbering
    double* d_val = nullptr;
    double* d_dinv = nullptr;             // Jacobi
    double gersh = 0.0;                   // Gershgorin bound of D^-1 A (all ranks)
    int64_t n_ghost = 0;
    int32_t* d_boundary_rows = nullptr;
    int64_t n_boundary = 0;
    int32_t* d_interior_rows = nullptr;
    int64_t n_interior = 0;
    int interior_contig = 1;
    int64_t interior_begin = 0;
    std::vector<bk_neighbor> nbs;
    int64_t n_send_total = 0;
    bk_buf ghost, sendbuf;
    bk::BandPlan band;                    // band plan of the contiguous interior range
};

// workspace slots used by the ABI and the solvers
enum bk_ws_slot {
    WS_STAGE_X = 0, WS_STAGE_Y, WS_STAGE_C, WS_STAGE_G, WS_GRAM_PART, WS_COLDOT_PART,
    WS_SOLVE_BASE  // solvers use WS_SOLVE_BASE + i
};

namespace bk {
void* ws_get(bk_ctx* ctx, int slot, size_t bytes);  // throws on OOM
int set_error(bk_ctx* ctx, int code, const std::string& msg);
int cuda_check(bk_ctx* ctx, cudaError_t e, const char* where);
bool is_device_ptr(const void* p);
int halo_exchange(bk_ctx* ctx, const bk_csr* A, int k, const double* X, int64_t ldx);
int allreduce_sum(bk_ctx* ctx, double* d, int64_t n);
// collective (nranks > 1): halo plan, renumbering, neighbour lists (comm.cpp)
int csr_setup_comm(bk_ctx* ctx, bk_csr* A, const std::vector<int32_t>& rp, std::vector<int32_t>& col_local,
                   const std::vector<int32_t>& colg);
// Y = A X with the fused reduction epilogue (launch_bspmm_win_red) on a single-rank matrix whose
// band plan allows it; false = not applicable (the caller runs the separate passes)
bool spmm_red_dev(bk_ctx* ctx, const bk_csr* A, int k, const double* X, double* Y, int red, const double* e0,
                  const double* e1, double* blk0, double* blk1, double* dot0, double* dot1, const SmallEpi* epi);
int solve_impl(bk_ctx* ctx, const bk_csr* A, int k, const double* B, int64_t ldb, double* X,
               int64_t ldx, const bk_solve_opts* o, bk_solve_report* rep);
int dirk_b0_impl(bk_ctx* ctx, const bk_csr* K, double mass, double tau, int m, const double* A, int s,
                 const double* yn, const double* bn, double* B0, int64_t ldb, double* scratch);
int dirk_impl(bk_ctx* ctx, const bk_csr* L, const bk_csr* K, double mass, double tau, int k, const double* A1h,
              const double* A2h, const double* B, const double* B0, int64_t ldb, double* Y, int64_t ldy,
              int max_outer, double outer_tol, const bk_solve_opts* inner, bk_dirk_report* rep, bool correction = false);
// device-pointer variants used by the solvers (no host staging, no validation)
int spmm_dev(bk_ctx* ctx, const bk_csr* A, int k, const double* X, int64_t ldx, const double* C,
             int kout, double alpha, double beta, double* Y, int64_t ldy);
int gram_dev(bk_ctx* ctx, int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y,
             int64_t ldy, double* G, bool allreduce);
}  // namespace bk

struct bk_error : std::exception {
    int code;
    std::string msg;
    bk_error(int c, std::string m) : code(c), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};
