/*
 * bk.h -- C ABI of the B200-native block-Krylov hot path of arxiv 2504.02117
 * ("vectorised DIRK time integration via block Krylov").
 *
 * The paper reformulates m DIRK stages x s time steps as ONE matrix equation
 * A X = B with k = s*m columns (§2.1, eq. (matrix-fixed-point-
 * equation)) and solves it with a vectorised block Krylov method
 * (Algorithm 1 "solve JV = R").  The solver's time is spent in the
 * block operator apply (BOP, §3), the k x k block inner products
 * and the block updates.  This library exports exactly those calls.
 *
 * Conventions (all entry points):
 *  - Values are IEEE float64; CSR indices int32 (nnz < 2^31); sizes int64.
 *  - Multivectors are ROW-MAJOR N x k with leading dimension ld >= k (all k
 *    entries of a row adjacent: the SIMD/lane axis of the paper).
 *  - Small matrices (C, G) are ROW-MAJOR and act as RIGHT multipliers, so the
 *    paper's "(A_2 - beta I)^T" is passed already transposed.
 *  - Pointers to multivectors and small matrices may be DEVICE memory (of the
 *    ctx's device) or HOST memory (pinned or pageable).  Device pointers make
 *    the call stream-ordered and asynchronous on the ctx stream.  Host pointers
 *    are staged through library-owned device buffers; the call then returns
 *    only after host outputs are written (synchronous).
 *  - The caller owns every buffer it passes; the library never frees or
 *    retains them after return.  bk_csr_create COPIES the matrix.
 *  - Argument/contract violations return BK_ERR_ARG before any work is
 *    enqueued; the message is available from bk_last_error(ctx).  CUDA/NCCL
 *    failures return BK_ERR_CUDA / BK_ERR_NCCL and are sticky for the ctx.
 *  - One ctx per host thread / stream.  Outputs must not alias inputs unless
 *    stated.  No CPU fallback exists: every numeric step runs in sm_100a kernels.
 */
#ifndef BK_H
#define BK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BK_MAX_K 32          /* max block width k of apply / update / solve  */
#define BK_MAX_KA 4096       /* max rows of a (multi-)Gram result            */

enum bk_status {
    BK_OK = 0,
    BK_ERR_ARG = 1,          /* invalid argument, nothing was enqueued       */
    BK_NOT_CONVERGED = 2,    /* solver hit max_iters (X = last iterate)      */
    BK_BREAKDOWN = 3,        /* singular k x k block (report.breakdown_column) */
    BK_ERR_CUDA = 4,
    BK_ERR_NCCL = 5,
    BK_ERR_OOM = 6,
    BK_ERR_UNSUPPORTED = 7
};

typedef struct bk_ctx bk_ctx;
typedef struct bk_csr bk_csr;

/* ---------------------------------------------------------------- context */
int         bk_version(void);                       /* e.g. 100 = 0.1.0      */
const char *bk_status_string(int status);
/* Message of the last failure on ctx (never NULL; "" if none).            */
const char *bk_last_error(const bk_ctx *ctx);
/* Number of CUDA kernels this library has launched in this process (all
 * contexts, monotonically increasing; for launch accounting in benchmarks). */
int64_t     bk_kernel_launch_count(void);

/* Create a context on CUDA device `device`, ordering work on `cuda_stream`
 * (a cudaStream_t, used as is; NULL = the legacy default stream).  The
 * stream stays owned by the caller.                                        */
int bk_ctx_create(bk_ctx **out, int device, void *cuda_stream);
int bk_ctx_set_stream(bk_ctx *ctx, void *cuda_stream);
int bk_ctx_synchronize(bk_ctx *ctx);
int bk_ctx_destroy(bk_ctx *ctx);

/* ---------------------------------------------------------------- multi-GPU
 * contiguous row partition (z-slabs for lexicographic grids);
 * halo rows exchanged with NCCL send/recv over NVLink, overlapped with the
 * interior rows; k x k Gram matrices summed with NCCL allreduce.
 * bk_get_nccl_unique_id: rank 0 fills 128 bytes, the caller broadcasts them
 * (e.g. torch.distributed) and every rank calls bk_ctx_set_comm collectively. */
int bk_get_nccl_unique_id(void *out128);
int bk_ctx_set_comm(bk_ctx *ctx, const void *uid128, int nranks, int rank);
int bk_ctx_comm_info(const bk_ctx *ctx, int *nranks, int *rank);

/* Loopback transport (TEST INFRASTRUCTURE for the row-partitioned path on a one-GPU box):
 * `nranks` virtual ranks live in ONE process, one host thread and one ctx each (any
 * devices, typically all on device 0).  bk_ctx_set_comm_local attaches a ctx as rank `rank`
 * of the hub instead of an NCCL communicator; every collective of the library
 * (bk_csr_create's halo-plan exchange, the halo exchange inside bspmm_apply, the Gram
 * allreduce, the solvers' reductions) then runs between host barriers with device-to-device
 * copies, reductions on the device in rank order -- the same protocol, the same
 * interior / boundary kernels, bitwise-identical results on every rank.  Every rank's thread
 * must make the same sequence of collective calls (as with NCCL).  The hub must outlive the
 * contexts attached to it; it holds no device memory.  Returns BK_OK or BK_ERR_ARG.      */
int bk_local_hub_create(void **hub, int nranks);
int bk_local_hub_destroy(void *hub);
int bk_ctx_set_comm_local(bk_ctx *ctx, void *hub, int rank);

/* ---------------------------------------------------------------- matrix
 * Local row slab [row_begin, row_begin + n_local) of an n_global x n_global
 * CSR matrix (SPEC S:26-31 invariants: row_ptr[0] = 0, non-decreasing,
 * row_ptr[n_local] = nnz, columns strictly increasing per row, GLOBAL column
 * ids in [0, n_global)).  Arrays may be host or device; they are copied (and
 * for nranks > 1 renumbered: local columns first, then ghost columns, and
 * split into interior/boundary rows).  For nranks > 1 the call is collective
 * (it exchanges the halo plan).  With a single rank, row_begin must be 0 and
 * n_local == n_global.                                                      */
int bk_csr_create(bk_ctx *ctx, bk_csr **out, int64_t n_global, int64_t row_begin,
                  int64_t n_local, const int32_t *row_ptr, const int32_t *col_global,
                  const double *val, int64_t nnz);
/* Destroying a ctx detaches its matrices (their handles stay valid for
 * bk_csr_destroy, which then only frees memory; any other use is an error). */
int bk_csr_destroy(bk_csr *A);

typedef struct bk_csr_info {
    int64_t n_global, row_begin, n_local, nnz;
    int64_t n_ghost;          /* ghost rows received per apply              */
    int64_t n_boundary_rows;  /* rows touching a ghost column               */
    int64_t n_send_rows;      /* rows sent to other ranks per apply         */
    int     n_neighbors;
    int     interior_contiguous; /* interior rows form one contiguous range */
    int     n_bands;          /* diagonal bands of the windowed apply
                                 (bk_plan_bands; 0: unstaged gathers)        */
    int     band_extra_rows;  /* window rows per tile beyond n_bands * T      */
    double  jacobi_gershgorin; /* max_i sum_j |a_ij| / |a_ii| (all ranks): an upper
                                  bound of the spectrum of D^-1 A (Chebyshev lmax) */
} bk_csr_info;
int bk_csr_get_info(const bk_csr *A, bk_csr_info *info);

/* ---------------------------------------------------------------- kernels */

/* a1: Block operator apply (BOP, §3; column independence
 * (I_m (x) A) vec X = vec(A X), §2.1; coupling term -K Y C with
 * C = (A_2 - beta I)^T of eq. (matrix-fixed-point-equation)):
 *
 *     Y = alpha * (A X) C + beta * Y
 *
 * X: n_local x k (ld ldx), the LOCAL slab only (ghost rows are fetched by the
 *    library with NCCL when nranks > 1).  1 <= k <= BK_MAX_K.
 * C: k x k_out row-major, or NULL for C = I (then k_out must equal k).
 * Y: n_local x k_out (ld ldy).  beta == 0: Y is not read.  Y must not alias X.
 * Streams the CSR once for all k columns.                      */
int bspmm_apply(bk_ctx *ctx, const bk_csr *A, int k, const double *X, int64_t ldx,
                const double *C, int k_out, double alpha, double beta,
                double *Y, int64_t ldy);

/* a3: Block Gram / block inner product (§1 P:43 "information
 * exchange between the columns"):  G = X^T Y,  G[a][b] = sum_i X[i,a] Y[i,b].
 * X: n x ka (ldx), Y: n x kb (ldy); 1 <= ka <= BK_MAX_KA, 1 <= kb <= BK_MAX_K.
 * G: ka x kb row-major (host or device).  Deterministic: fixed-order two-stage
 * reduction, bitwise reproducible run to run.  flags & BK_GRAM_ALLREDUCE sums
 * G over the ctx's ranks (NCCL allreduce) -- every rank gets identical bits. */
#define BK_GRAM_ALLREDUCE 1
int block_gram(bk_ctx *ctx, int64_t n, int ka, int kb, const double *X, int64_t ldx,
               const double *Y, int64_t ldy, double *G, int flags);

/* a5: Block update (block axpy of the Krylov recurrences; the splitting RHS
 * terms B A_2^T, -M Y (A_1 - I/tau)^T of P:389-395 with M = h^d I):
 *
 *     X = a * X + s * P C
 *
 * X: n x k (ldx), P: n x kp (ldp), C: kp x k row-major (host or device).
 * 1 <= k <= BK_MAX_K, 1 <= kp <= BK_MAX_KA.  a == 0: X is not read.
 * P may alias X only when P == X, ldp == ldx and kp == k (in-place X C).    */
int block_update(bk_ctx *ctx, int64_t n, int kp, int k, double a, double *X, int64_t ldx,
                 double s, const double *P, int64_t ldp, const double *C);

/* a6: Block Krylov solve of A X = B (Algorithm 1 "solve
 * JV = R"; DUNE-ISTL Block-CG / Block-BiCGStab P:932-934, P:1054-1056,
 * P:1346-1348; O'Leary block CG P:43).  X holds X0 on entry (ignored when
 * opts->x0_is_zero) and the last iterate on return.  Convergence: every column
 * ||B_c - (A X)_c||_2 <= rtol ||B_c - (A X0)_c||_2 ("defect reduction
 * ... for all right-hand-sides"), using the method's recurrence residual;
 * rep->true_relres is recomputed from scratch at the end.
 * Returns BK_OK, BK_NOT_CONVERGED or BK_BREAKDOWN (also in rep->status).   */
/* BK_CG1 (the communication-avoiding form the paper's P:43
 * motivates): single-reduction block CG -- the O'Leary iterates (in exact arithmetic) with
 * every k x k quantity of an iteration taken from ONE reduction pass over [R, W = A R]
 * (Q = A P by recurrence; one allreduce per iteration for nranks > 1); SPD A,
 * unpreconditioned (R32, oracle O11).                                           */
enum bk_method  { BK_CG = 0, BK_GMRES = 1, BK_BICGSTAB = 2, BK_CG1 = 3 };
/* Preconditioners (CG only: M^-1 must be SPD).  CHEBYSHEV (SURVEY.md §8(f) NEXT-4,
 * the polynomial stand-in for the paper's AMG preconditioner):
 * M^-1 R = cheb_steps steps of Chebyshev acceleration (Saad Alg. 12.1) for A Z = R
 * from Z = 0 with the Jacobi splitting on [cheb_lmin, cheb_lmax]:
 * Z = p(D^-1 A) D^-1 R, deg p = cheb_steps - 1 (cheb_steps - 1 applies per use).
 * cheb_lmax <= 0: the Gershgorin bound (bk_csr_info.jacobi_gershgorin);
 * cheb_lmin <= 0: cheb_lmax / 30 (R28).  SPD for SPD A whenever
 * cheb_lmax bounds the spectrum of D^-1 A.                                       */
enum bk_precond { BK_PRECOND_NONE = 0, BK_PRECOND_JACOBI = 1, BK_PRECOND_CHEBYSHEV = 2 };
enum bk_conv    { BK_CONV_ALL = 0, BK_CONV_FIRST = 1 };

typedef struct bk_solve_opts {
    int    method;          /* enum bk_method                                 */
    int    max_iters;       /* block iterations (GMRES: inner steps, total)   */
    int    restart;         /* GMRES(m): m >= 1                               */
    int    precond;         /* enum bk_precond (JACOBI, CHEBYSHEV: CG only)   */
    int    conv_mode;       /* enum bk_conv                                   */
    int    x0_is_zero;      /* 1: ignore X on entry                           */
    int    check_every;     /* host-side convergence poll period (>= 1)       */
    int    use_graphs;      /* 1: CG / BiCGStab iterations replayed from a CUDA
                               graph captured once per solve (one rank, timing
                               off; GMRES ignores it) -- for small, launch-bound
                               systems                                        */
    double rtol;
    double breakdown_tol;   /* relative pivot threshold (default 1e-13)       */
    int    timing;          /* 1: CUDA events around every N x k kernel on the
                               ctx stream -> rep->t_class_ms / n_class       */
    int    cheb_steps;      /* CHEBYSHEV: steps (>= 1; default 4)             */
    double cheb_lmin;       /* CHEBYSHEV interval (<= 0: defaults, above)     */
    double cheb_lmax;
} bk_solve_opts;

/* NEXT-4: Z = M^-1 R for the preconditioner opts->precond of A (NONE: copy;
 * JACOBI: D^-1 R; CHEBYSHEV: as above).  R, Z: n_local x k row-major, host or
 * device, Z must not alias R.  Collective for nranks > 1 (the Chebyshev applies
 * exchange halos).  Returns BK_OK or an error code.                               */
int bk_precond_apply(bk_ctx *ctx, const bk_csr *A, int k, const bk_solve_opts *opts, const double *R,
                     int64_t ldr, double *Z, int64_t ldz);

/* kernel classes of bk_solve_report.t_class_ms / n_class */
enum bk_kclass { BK_K_SPMM = 0, BK_K_GRAM = 1, BK_K_UPDATE = 2, BK_K_FUSED_TAIL = 3,
                 BK_K_FUSED_GRAM = 4 /* Rt^T [V R] */, BK_K_COPY = 5,
                 BK_K_FUSED_DOTS = 6 /* Rt^T T, <T,S>, <T,T> */,
                 BK_K_FUSED_APPLY = 7 /* apply with k x k Gram blocks in its epilogue (Rt^T [V R],
                                         P^T Q, [R^T W, R^T R]) */,
                 BK_K_FUSED_APPLY_DOTS = 8 /* apply with Rt^T T, <T,S>, <T,T> in its epilogue */,
                 BK_NKCLASS = 9 };

typedef struct bk_solve_report {
    int     status;           /* BK_OK / BK_NOT_CONVERGED / BK_BREAKDOWN      */
    int     iterations;
    int     converged;
    int     breakdown_column; /* -1 if none                                   */
    double  relres[BK_MAX_K];      /* recurrence residual / initial, per column */
    double  true_relres[BK_MAX_K]; /* ||B - A X|| / initial, recomputed       */
    double  t_total_ms;
    int64_t n_spmm, n_gram, n_update, n_small, n_allreduce;
    double  t_class_ms[BK_NKCLASS];  /* opts->timing: summed event time per kernel class */
    int64_t n_class[BK_NKCLASS];     /* launches timed per class                        */
    int64_t alg_bytes;        /* ALGORITHMIC bytes of every N x k pass and apply this
                                 call enqueued (CSR streamed once, each operand read /
                                 written once per pass): the numerator of
                                 the solver's GB/s, counted where the passes are issued */
} bk_solve_report;

void bk_solve_opts_default(bk_solve_opts *opts);

int block_krylov_solve(bk_ctx *ctx, const bk_csr *A, int k, const double *B, int64_t ldb,
                       double *X, int64_t ldx, const bk_solve_opts *opts,
                       bk_solve_report *rep);

/* ---------------------------------------------------------------- NEXT-1: DIRK window
 * s time steps x m stages of a stiffly accurate DIRK method as ONE matrix equation
 * with k = s m columns (§2.1, eq. general-system-time-steps P:104-126,
 * window matrices P:260-288):
 *     M Y A1^T + K Y A2^T = B A2^T + B0,          M = mass * I,
 * solved by the splitting fixed point (eq. matrix-splitting / matrix-fixed-point-
 * equation), beta = A2[0][0], L = M/tau + beta K:
 *     L Y^j = -M Y^{j-1} (A1 - I/tau)^T - K Y^{j-1} (A2 - beta I)^T + B A2^T + B0,
 * one block_krylov_solve per outer iteration (opts `inner`, started from zero:
 * a warm start leaves already-exact columns with a zero residual, on which the
 * block method breaks down -- no deflation).  For SDIRK windows both couplings are strictly lower triangular, so
 * the iteration is exact after k outer steps (column c after c + 1), up to the
 * inner tolerance.
 * L, K: matrices of the same row partition (L must equal M/tau + beta K; the
 *   caller assembles it).  A1, A2: k x k row-major, HOST.  B, B0: N x k (ld ldb),
 *   host or device.  Y: N x k (ld ldy): Y^0 on entry, the last iterate on return.
 * outer_tol > 0: stop when ||Y^j - Y^{j-1}||_F <= outer_tol ||Y^j||_F;
 *   0: run max_outer iterations.
 * Returns BK_OK, BK_NOT_CONVERGED or BK_BREAKDOWN (of an inner solve; also in
 * rep->status), or an error status.                                          */
typedef struct bk_dirk_report {
    int    status;
    int    outer_iterations;
    int    inner_iterations_total;
    int    last_inner_status;
    double last_change;      /* ||Y^j - Y^{j-1}||_F / ||Y^j||_F, last outer step */
    double t_total_ms;
} bk_dirk_report;
int bk_dirk_solve(bk_ctx *ctx, const bk_csr *L, const bk_csr *K, double mass, double tau, int k,
                  const double *A1, const double *A2, const double *B, const double *B0, int64_t ldb,
                  double *Y, int64_t ldy, int max_outer, double outer_tol,
                  const bk_solve_opts *inner, bk_dirk_report *rep);
/* Same window equation in defect-correction form (the paper's outer / inner tolerance policy
 * for s > 1, §4.1: a loose inner tolerance, the outer iterations refresh the
 * right-hand side): per outer iteration F = B A2^T + B0 - M Y (A1 - I/tau)^T ... - L Y is the
 * defect of the split system, L D = F is solved from D = 0 to inner->rtol (columns scaled to
 * unit norm; a block breakdown falls back to column-wise solves), Y += D.  Stops when
 * ||F||_F / ||F_0||_F <= outer_tol (rep->last_change) or after max_outer iterations.
 * Y holds the initial guess.  Arguments, ownership and errors as bk_dirk_solve.            */
int bk_dirk_solve_dc(bk_ctx *ctx, const bk_csr *L, const bk_csr *K, double mass, double tau, int k,
                     const double *A1, const double *A2, const double *B, const double *B0, int64_t ldb,
                     double *Y, int64_t ldy, int max_outer, double outer_tol,
                     const bk_solve_opts *inner, bk_dirk_report *rep);

/* Window matrices of NEXT-1 from a Butcher tableau (host only, no GPU; §2.1): s
 * consecutive time steps of the diagonally implicit, stiffly accurate tableau A (m x m,
 * row-major, lower triangular, c = A 1) as one matrix equation with k = s m' columns
 * (R24): A2 = I_s (x) A', A1 = I / tau, A1[q m' + i][q m' - 1] = -1/tau
 * for q >= 1.  An explicit first stage (a_11 = 0, e.g. the Theta-method) is eliminated first
 * (P:128-213): A' = A[1:, 1:], m' = m - 1, and its column a_{i1} couples each step to the
 * previous step's last stage: A2[q m' + i][q m' - 1] = a_{i+1,1} for q >= 1 (the
 * q = 0 coupling is the B0 term of bk_dirk_b0).  Only the first stage may be explicit.
 * A1, A2: caller-allocated k x k (k <= BK_MAX_K) row-major, overwritten.  a_elim: NULL or m'
 * doubles, receives (a_21, ..., a_m1) (zeros without an eliminated stage).  *k_out = k.
 * Returns BK_OK or BK_ERR_ARG (not DIRK, a later explicit stage, tau <= 0, k > 32).          */
int bk_dirk_window(int m, const double *A, int s, double tau, int *k_out, double *A1, double *A2,
                   double *a_elim);
/* B0 of that window, computed on the device: column i < m' equals
 * (mass / tau) y^n + a_{i+1,1} (b^n - K y^n) (the second term only for an eliminated explicit
 * first stage; one apply of K), the other columns are 0.  K: the stiffness matrix (same
 * partition as the window's unknowns; collective for nranks > 1).  y^n, b^n: n_local doubles
 * (host or device; b^n may be NULL = 0).  B0: n_local x k (ld ldb >= k), host or device,
 * overwritten.  Returns BK_OK or an error status.                                          */
int bk_dirk_b0(bk_ctx *ctx, const bk_csr *K, double mass, double tau, int m, const double *A, int s,
               const double *yn, const double *bn, double *B0, int64_t ldb);

/* NEXT-3: Algorithm 1 "Block Krylov Time Stepping with Pipelining" (§2.2
 * P:600-621; eq. matrix-equation-pipelining; shift P:592-594; iota P:574-580)
 * on the nonlinear diffusion-reaction problem M y' + f(t, y) = 0 of an nx x ny x nz
 * cell-centred lattice (x fastest; h = 1/nx; M = h^3 I; Neumann; R29):
 *   f(t,u)_a = sum_b h D_ab (u_a - u_b) + h^3 (u_a - u_a^2) - h^3 sin(1 + t) g_a,
 *   D_ab = 1 + (u_a^2 + u_b^2)/2,
 * stepped with the stiffly accurate DIRK tableau A (m x m row-major, host; c = A 1),
 * t^n = n tau, a pipelined window of `window` consecutive stages.  Per stage: shift;
 * Newton loop: R = M Y A1^T + F(T,Y) A2^T - B0 (sign reading R30); stop when
 * ||R_0||_2 < eps; J = M/tau + a_kk Df(t, Y_0) assembled on the device; solve J V = R
 * with block_krylov_solve(inner, x0 = 0, k = window); Y -= V.
 * y0, g: N = nx ny nz doubles (host or device).  traj: N x n_steps row-major with
 * leading dimension ldt >= n_steps (host or device; column n = y^{n+1}), may be NULL.
 * newton_its: host int[n_steps * m] (Newton iterations per accepted stage) or NULL.
 * Single rank only (nranks == 1).  Returns BK_OK, BK_NOT_CONVERGED (a stage needed
 * more than max_newton iterations; rep->failed_stage) or an error status.           */
typedef struct bk_dr_problem {
    int64_t nx, ny, nz;
    double  tau;
    const double *y0;
    const double *g;
} bk_dr_problem;
typedef struct bk_alg1_report {
    int    status;
    int    stages_accepted;
    int    newton_iterations_total;
    int    inner_iterations_total;
    int    inner_breakdowns;
    int    failed_stage;
    double last_norm;
    double t_total_ms;
} bk_alg1_report;
int bk_alg1_run(bk_ctx *ctx, const bk_dr_problem *prob, int m, const double *A, int n_steps, int window,
                double eps, int max_newton, const bk_solve_opts *inner, double *traj, int64_t ldt,
                int *newton_its, bk_alg1_report *rep);

/* ---------------------------------------------------------------- host-only
 * Halo plan of a contiguous row partition (pure host code, no CUDA; exported
 * for CPU tests of the multi-GPU path).  Given this rank's local CSR columns
 * (global ids) and the partition bounds rank_begin[0..nranks] (rank r owns
 * rows [rank_begin[r], rank_begin[r+1])), computes:
 *   ghost_ids[n_ghost]   sorted global ids of non-local columns,
 *   ghost_owner[n_ghost] owning rank of each,
 *   col_local[nnz]       renumbered columns: local j -> j - row_begin,
 *                        ghost g -> n_local + (index of g in ghost_ids),
 *   is_boundary[n_local] 1 if the row touches a ghost column.
 * Output arrays are caller-allocated (ghost arrays sized nnz for safety).
 * Returns BK_OK or BK_ERR_ARG.                                              */
int bk_plan_halo(int nranks, int rank, const int64_t *rank_begin,
                 int64_t n_local, const int32_t *row_ptr, const int32_t *col_global,
                 int64_t nnz, int64_t *n_ghost, int64_t *ghost_ids, int32_t *ghost_owner,
                 int32_t *col_local, uint8_t *is_boundary);

/* Band plan of the windowed apply (pure host code, run by
 * bk_csr_create on the contiguous (interior) row range, exported for CPU
 * tests).  The paper's BOP streams the matrix once for all k columns
 * (P:666-667); on B200 the X rows a tile of rows needs are moved into shared
 * memory by TMA bulk copies so the gathers become shared-memory loads.  For a
 * structured-grid operator every nonzero lies on a few diagonals d = col - row
 * (5-point: 0, +-1, +-nx; 7-point: also +-nx*ny).  The distinct offsets are
 * merged into BANDS (gaps <= 4); band g = offsets [dmin, dmax].  For a tile of
 * rows [r0, r0 + T) (r0, T even) band g needs X rows [r0 + lo, r0 + T + hi)
 * with lo = dmin rounded down and hi = dmax + 1 rounded up to even (16-byte
 * aligned TMA copies for any k).  The matrix is band structured (nbands > 0)
 * when there are <= BK_BAND_MAX bands and sum(hi - lo) <= max_extra;
 * otherwise nbands = 0 and the apply uses the unstaged gather kernel.
 * row_ptr: n_rows + 1 offsets into col (any base); row i of the range has
 * local index i (d = col - i).  Returns BK_OK or BK_ERR_ARG.                */
#define BK_BAND_MAX 7
typedef struct bk_band_plan {
    int32_t nbands;                 /* 0 = not band structured               */
    int32_t extra_rows;             /* sum(hi - lo): window = nbands*T + this */
    int32_t max_row_nnz;            /* sum of band widths (>= nnz of any row) */
    int32_t dmin[BK_BAND_MAX], dmax[BK_BAND_MAX], width[BK_BAND_MAX];
    int32_t lo[BK_BAND_MAX], hi[BK_BAND_MAX];
} bk_band_plan;
int bk_plan_bands(int64_t n_rows, const int32_t *row_ptr, const int32_t *col, int max_extra,
                  bk_band_plan *out);

#ifdef __cplusplus
}
#endif
#endif /* BK_H */
