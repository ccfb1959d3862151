/*
 * bk_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously correct definitions of the three N x k operations on
 * the hot path of arxiv 2504.02117 (vectorised DIRK via block Krylov).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header, table or
 * helper with the CUDA path (paper_2504_02117_b200/) and includes none of it.
 *
 * Compiled with gcc -O2 -ffp-contract=off (no FMA contraction, no fast-math),
 * single threaded.  Every function cites the passage it writes out.
 *
 *   PAPER.md = /root/reference/PAPER.md ("P:n" = line n), SPEC.md ("S:n").
 */
#include <stdint.h>
#include <stddef.h>

/*
 * O1  Block operator apply (BOP, §3 P:660-664 "Y <- A X";
 *     column independence (I_m (x) A) vec X = vec(A X), §2.1 P:338-356;
 *     the k x k coupling "- K Y (A_2 - beta I)^T" of eq. (matrix-fixed-point-
 *     equation) P:389-395 is a right multiplier C).
 *
 *     Y = alpha * (A X) C + beta * Y
 *
 * For each row i ascending:  t[c] = sum_p val[p] * X[col[p], c] in CSR order,
 * separate multiply and add; u[c'] = sum_c t[c] * C[c, c'] (c ascending;
 * C == NULL means C = I, u = t); Y[i, c'] = alpha*u[c'] + beta*Y[i, c'].
 * beta == 0: Y is not read (NaN garbage is overwritten).  C is row-major
 * k x k_out.  k <= 64 (local accumulator).
 */
int oracle_spmm(int64_t n_rows, const int32_t *row_ptr, const int32_t *col,
                const double *val, int k, const double *X, int64_t ldx,
                const double *C, int k_out, double alpha, double beta,
                double *Y, int64_t ldy)
{
    if (k < 1 || k > 64 || k_out < 1 || k_out > 64) return 1;
    if (C == NULL && k_out != k) return 1;
    for (int64_t i = 0; i < n_rows; ++i) {
        double t[64], u[64];
        for (int c = 0; c < k; ++c) t[c] = 0.0;
        for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const double *xr = X + (int64_t)col[p] * ldx;
            for (int c = 0; c < k; ++c) {
                double prod = val[p] * xr[c];
                t[c] = t[c] + prod;
            }
        }
        if (C != NULL) {
            for (int co = 0; co < k_out; ++co) {
                double s = 0.0;
                for (int c = 0; c < k; ++c) {
                    double prod = t[c] * C[(int64_t)c * k_out + co];
                    s = s + prod;
                }
                u[co] = s;
            }
        } else {
            for (int c = 0; c < k; ++c) u[c] = t[c];
        }
        double *yr = Y + i * ldy;
        for (int co = 0; co < k_out; ++co) {
            double a = alpha * u[co];
            if (beta != 0.0) {
                double b = beta * yr[co];
                yr[co] = a + b;
            } else {
                yr[co] = a;
            }
        }
    }
    return 0;
}

/* O1 on a subset of rows (sampled parity at full size: SpMM rows are
 * independent, so each selected row is the plain definition above).
 * Y_sel is n_sel x k_out row-major; beta is applied to Y_sel's input. */
int oracle_spmm_rows(const int64_t *rows, int64_t n_sel, const int32_t *row_ptr,
                     const int32_t *col, const double *val, int k,
                     const double *X, int64_t ldx, const double *C, int k_out,
                     double alpha, double beta, double *Y_sel)
{
    for (int64_t s = 0; s < n_sel; ++s) {
        int64_t i = rows[s];
        int32_t rp[2] = {0, row_ptr[i + 1] - row_ptr[i]};
        int r = oracle_spmm(1, rp, col + row_ptr[i], val + row_ptr[i], k, X, ldx,
                            C, k_out, alpha, beta, Y_sel + s * k_out, k_out);
        if (r) return r;
    }
    return 0;
}

/*
 * O2  Block Gram / block inner product G = X^T Y (§1, the k x k
 *     block inner products through which the columns "exchange information";
 *     SPEC dot_columns S:71-79).  G[a][b] = sum_i X[i,a] * Y[i,b], each
 *     product exact-rounded, accumulated in long double (x87, 64-bit
 *     mantissa) in row order, rounded once to double.  G is ka x kb row-major.
 */
int oracle_gram(int64_t n, int ka, int kb, const double *X, int64_t ldx,
                const double *Y, int64_t ldy, double *G)
{
    if (ka < 1 || kb < 1) return 1;
    for (int a = 0; a < ka; ++a) {
        for (int b = 0; b < kb; ++b) {
            long double s = 0.0L;
            for (int64_t i = 0; i < n; ++i) {
                long double prod = (long double)X[i * ldx + a] * (long double)Y[i * ldy + b];
                s = s + prod;
            }
            G[(int64_t)a * kb + b] = (double)s;
        }
    }
    return 0;
}

/*
 * O3  Block update X <- a*X + s*P*C (block axpy of the Krylov recurrences;
 *     also the splitting RHS terms B A_2^T and -M Y (A_1 - I/tau)^T of
 *     eq. (matrix-fixed-point-equation) P:389-395 with M = h^d I).
 *     X[i,b] = a*X[i,b] + s * sum_{c ascending} P[i,c] * C[c,b]; a == 0: X not read.
 *     C is kp x k row-major.
 */
int oracle_update(int64_t n, int kp, int k, double a, double *X, int64_t ldx,
                  double s, const double *P, int64_t ldp, const double *C)
{
    if (kp < 1 || k < 1) return 1;
    for (int64_t i = 0; i < n; ++i) {
        for (int b = 0; b < k; ++b) {
            double acc = 0.0;
            for (int c = 0; c < kp; ++c) {
                double prod = P[i * ldp + c] * C[(int64_t)c * k + b];
                acc = acc + prod;
            }
            double sv = s * acc;
            if (a != 0.0) {
                double av = a * X[i * ldx + b];
                X[i * ldx + b] = av + sv;
            } else {
                X[i * ldx + b] = sv;
            }
        }
    }
    return 0;
}
