"""Algorithmic traffic / flop counts and the paper's performance model (host logic only).

* Paper (context): AI(spMV) = 1/8 (§1); AI(spBOP) = k / (4 (k+1))
  (§3, Fig. AIBOP); simplified ECM counts omega = 2kz FLOP,
  beta = 2z + 2kz doubles, tau = z (2 + 2k) doubles (§3).
* Algorithmic bytes (what the method must move): the CSR streamed
  once, every multivector read once and written once.  These are the numerators
  of every GB/s this repo reports (bench.py `roofline.achieved`).
"""
from __future__ import annotations

from fractions import Fraction

D = 8   # bytes per float64
I = 4   # bytes per int32


# ------------------------------------------------------------------ paper model
def paper_ai_spmv() -> Fraction:
    """two FLOP per two doubles -> 1/8 FLOP/byte."""
    return Fraction(2, 2 * D)


def paper_ai_spbop(k: int) -> Fraction:
    """2k FLOP per (k + 1) doubles -> k / (4 (k+1)) FLOP/byte."""
    return Fraction(2 * k, (k + 1) * D)


def paper_ecm_counts(k: int, z: int):
    """(omega FLOP, beta doubles from memory, tau doubles L1<->registers)."""
    return 2 * k * z, 2 * z + 2 * k * z, z * (2 + 2 * k)


# ------------------------------------------------------------------ algorithmic model
def spmm_bytes(n_rows: int, nnz: int, k: int, k_out: int | None = None, beta_nonzero: bool = False,
               n_ghost: int = 0) -> int:
    """12 nnz + 4 (N + 1) [CSR] + 8 k (N + N_ghost) [X read once] + 8 k_out N [Y write] (+ Y read if beta)."""
    k_out = k if k_out is None else k_out
    b = (I + D) * nnz + I * (n_rows + 1) + D * k * (n_rows + n_ghost) + D * k_out * n_rows
    if beta_nonzero:
        b += D * k_out * n_rows
    return b


def spmm_flops(nnz: int, k: int, n_rows: int = 0, k_out: int | None = None, coupled: bool = False) -> int:
    """2 nnz k (+ 2 N k k_out for the k x k_out coupling)."""
    f = 2 * nnz * k
    if coupled:
        f += 2 * n_rows * k * (k if k_out is None else k_out)
    return f


def gram_bytes(n: int, ka: int, kb: int, same: bool = False) -> int:
    """8 N (ka + kb); 8 N k for X^T X."""
    return D * n * (ka if same else ka + kb)


def gram_flops(n: int, ka: int, kb: int) -> int:
    return 2 * n * ka * kb


def update_bytes(n: int, kp: int, k: int, a_nonzero: bool = True, extra_term: bool = False) -> int:
    """8 N (kp + k) + 8 N k [X read if a != 0] (+ 8 N k for a third operand W)."""
    return D * n * (kp + k + (k if a_nonzero else 0) + (k if extra_term else 0))


def update_flops(n: int, kp: int, k: int) -> int:
    return 2 * n * kp * k


def coldot_bytes(n: int, k: int, n_y: int = 1) -> int:
    """Column dots of X with n_y other arrays (n_y = 0: ||X_c||^2, X read once)."""
    return D * n * k * (1 + n_y)


def bicgstab_fused(k: int) -> bool:
    """Whether solve.cpp takes the fused BiCGStab passes (k % 4 == 0, k <= 16)."""
    return k % 4 == 0 and k <= 16


def bicgstab_iter_bytes(n: int, nnz: int, k: int, fused: bool | None = None, fused_apply: bool = False) -> int:
    """One block BiCGStab iteration as enqueued by solve.cpp (DESIGN.md §3 O6, §4.4).

    Fused (default where solve.cpp fuses): 2 applies + [Rt V R] Gram pass (3 N x k reads)
    + S = R - V alpha (2 reads, 1 write) + [Rt S T] Gram pass (3 reads) + the tail
    X, R, P update with ||R|| (5 reads, 3 writes) = 17 N x k passes + 2 applies (+ 2 reads
    for the separate <T,S>, <T,T> pass when k does not divide 32)."""
    if fused is None:
        fused = bicgstab_fused(k)
    if fused and fused_apply:
        # one rank, 2-D band plan, k = 8 / 12 / 16 (solve.cpp fapply): Rt^T [V R] rides in the V = A P
        # apply (+ Rt, R read), Rt^T T, <T,S>, <T,T> in the T = A S apply (+ Rt read; S, T are the
        # apply's own operands): 2 applies + 14 N x k passes
        v = 8 * n * k
        return 2 * spmm_bytes(n, nnz, k) + 2 * v + v + update_bytes(n, k, k) + 8 * v
    if fused:
        v = 8 * n * k
        dots = 0 if 32 % k == 0 else coldot_bytes(n, k, 1)   # <T,S>, <T,T> in their own pass (T, S read)
        return 2 * spmm_bytes(n, nnz, k) + 3 * v + update_bytes(n, k, k) + 3 * v + 8 * v + dots
    b = 2 * spmm_bytes(n, nnz, k)                     # V = A P, T = A S
    b += 3 * gram_bytes(n, k, k)                      # Rt^T V, Rt^T R, Rt^T T
    b += coldot_bytes(n, k, 1) + coldot_bytes(n, k, 0)  # <T,S>, <T,T> (T, S read); ||R|| (R read)
    b += update_bytes(n, k, k)                        # S = R - V alpha
    b += update_bytes(n, k, k, extra_term=True)       # X += P alpha + omega S
    b += update_bytes(n, 0, k, extra_term=True)       # R = S - omega T
    b += update_bytes(n, 0, k, extra_term=True)       # Tmp = P - omega V
    b += update_bytes(n, k, k)                        # P = R + Tmp beta
    return b


def cg_iter_bytes(n: int, nnz: int, k: int, fused: bool | None = None, fused_apply: bool = False) -> int:
    """One block CG iteration (unpreconditioned) as enqueued by solve.cpp (O4).  Fused (k % 4 == 0, <= 16):
    apply + P^T Q (2 reads) + tail X, P, R, Q -> X, R with R^T R (4 reads, 2 writes) + P update.
    fused_apply (one rank, 2-D band plan, k = 8 / 12 / 16): P^T Q rides in the apply's epilogue."""
    if fused is None:
        fused = k % 4 == 0 and k <= 16
    if fused and fused_apply:
        v = 8 * n * k
        return spmm_bytes(n, nnz, k) + 6 * v + update_bytes(n, k, k)
    if fused:
        v = 8 * n * k
        return spmm_bytes(n, nnz, k) + 2 * v + 6 * v + update_bytes(n, k, k)
    return (spmm_bytes(n, nnz, k) + gram_bytes(n, k, k) + 2 * update_bytes(n, k, k)
            + gram_bytes(n, k, k, same=True) + update_bytes(n, k, k))


def cg1_iter_bytes(n: int, nnz: int, k: int, fused: bool | None = None, fused_apply: bool = False) -> int:
    """One single-reduction block CG iteration (O11) as enqueued by solve.cpp.  Fused (k % 4 == 0,
    <= 16): tail X, R, P, W, Q -> X, R, P, Q (5 reads, 4 writes) + W = A R with [R^T W, R^T R]
    (fused_apply: in the apply's epilogue, R read once from the staged window; else one Gram
    pass over R, W).  Unfused: four updates + the apply + the Gram pass (k <= 16)."""
    if fused is None:
        fused = k % 4 == 0 and k <= 16
    v = 8 * n * k
    red = 0 if fused_apply else 2 * v
    if fused:
        return 9 * v + spmm_bytes(n, nnz, k) + red
    return 4 * update_bytes(n, k, k) + spmm_bytes(n, nnz, k) + red


def gmres_step_bytes(n: int, nnz: int, k: int, j: int) -> int:
    """Inner step j (0-based) of block GMRES with BCGS2 + CholQR2 (O5)."""
    ka = (j + 1) * k
    b = spmm_bytes(n, nnz, k)
    b += 2 * (gram_bytes(n, ka, k) + update_bytes(n, ka, k))
    b += 2 * (gram_bytes(n, k, k, same=True) + update_bytes(n, k, k, a_nonzero=False))
    return b


def bicgstab_solve_bytes(n: int, nnz: int, k: int, iters: int, x0_is_zero: bool = True, rt_is_b: bool = True,
                         fused: bool | None = None, fused_apply: bool = False) -> int:
    """A whole block_krylov_solve(method=bicgstab) call as solve.cpp enqueues it (no convergence
    before `iters`).  X0 = 0 with a packed B (rt_is_b): R0 = P0 = Rt = B are read in place -- only
    ||R_c|| (one same-operand column-dot pass over B); otherwise R = B (copy; + an apply when
    X0 != 0), Rt = R0 (copy), P = R (copy), ||R_c||.  Then `iters` iterations and the final true
    residual (copy + apply with beta != 0 + ||.||)."""
    v = D * n * k
    if x0_is_zero and rt_is_b:
        b = coldot_bytes(n, k, 0)
    else:
        b = 2 * v + (0 if x0_is_zero else spmm_bytes(n, nnz, k, beta_nonzero=True))
        b += 2 * v + 2 * v + coldot_bytes(n, k, 0)
    b += iters * bicgstab_iter_bytes(n, nnz, k, fused, fused_apply)
    b += 2 * v + spmm_bytes(n, nnz, k, beta_nonzero=True) + coldot_bytes(n, k, 0)
    return b
