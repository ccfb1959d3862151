"""CPU ORACLE for the block-Krylov hot path of arxiv 2504.02117.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  It shares no code with the CUDA
product path (paper_2504_02117_b200/) and imports nothing from it; the only
module both sides use is ``synth`` (seeded inputs, no method arithmetic).

* ``bk_oracle.c`` (plain C, gcc -O2 -ffp-contract=off): O1 spmm, O2 gram
  (long-double accumulation), O3 update -- the plain definitions.
* this file: ctypes marshalling for those, and the block Krylov algorithms O4
  (block CG), O5 (block GMRES(m), BCGS2 + CholQR2), O6 (block BiCGStab), written
  step by step in float64 numpy with numpy/LAPACK for the k x k steps, plus
  O7 (dense reference solve) and O8 (the DIRK window of SURVEY.md §8(f) NEXT-1:
  sequential SDIRK stepping, the all-at-once Kronecker solve, the splitting
  fixed point), O9 (the Chebyshev polynomial preconditioner and
  its Gershgorin interval), O11 (single-reduction block CG).  SURVEY.md §8(c) and DESIGN.md §3 give the
  readings.  Pins live in tests/test_oracle_*.py.

Parity status: every function here is pinned (see DESIGN.md §3 table).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bk_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_spmm.argtypes = [I64, P, P, P, I32, P, I64, P, I32, D, D, P, I64]
        lib.oracle_spmm_rows.argtypes = [P, I64, P, P, P, I32, P, I64, P, I32, D, D, P]
        lib.oracle_gram.argtypes = [I64, I32, I32, P, I64, P, I64, P]
        lib.oracle_update.argtypes = [I64, I32, I32, D, P, I64, D, P, I64, P]
        for f in (lib.oracle_spmm, lib.oracle_spmm_rows, lib.oracle_gram, lib.oracle_update):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None else None


def _np(t, dtype):
    """Accept numpy arrays or CPU torch tensors; returns a C-contiguous numpy array."""
    if hasattr(t, "detach"):
        t = t.detach().cpu().numpy()
    return np.ascontiguousarray(t, dtype=dtype)


class CsrNp:
    """CSR as numpy arrays (int32 row_ptr/col, float64 val)."""

    def __init__(self, n_rows, n_cols, row_ptr, col, val):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr = _np(row_ptr, np.int32)
        self.col = _np(col, np.int32)
        self.val = _np(val, np.float64)

    @classmethod
    def of(cls, A):
        if isinstance(A, CsrNp):
            return A
        return cls(A.n_rows, A.n_cols, A.row_ptr, A.col, A.val)

    def diag(self):
        d = np.zeros(self.n_rows)
        for i in range(self.n_rows):
            for p in range(self.row_ptr[i], self.row_ptr[i + 1]):
                if self.col[p] == i:
                    d[i] += self.val[p]
        return d


# --------------------------------------------------------------------------- O1..O3
def spmm(A, X, C=None, alpha=1.0, beta=0.0, Y=None):
    """O1: Y = alpha (A X) C + beta Y (bk_oracle.c oracle_spmm)."""
    A = CsrNp.of(A)
    X = _np(X, np.float64)
    k = X.shape[1]
    Cn = None if C is None else _np(C, np.float64)
    k_out = k if Cn is None else Cn.shape[1]
    if Y is None:
        Y = np.zeros((A.n_rows, k_out))
    else:
        Y = _np(Y, np.float64).copy()
    r = _load().oracle_spmm(A.n_rows, _ptr(A.row_ptr), _ptr(A.col), _ptr(A.val), k, _ptr(X), k,
                            _ptr(Cn), k_out, float(alpha), float(beta), _ptr(Y), k_out)
    if r:
        raise ValueError("oracle_spmm: bad arguments")
    return Y


def spmm_rows(A, rows, X, C=None, alpha=1.0, beta=0.0, Y_sel=None):
    """O1 restricted to `rows` (returns len(rows) x k_out)."""
    A = CsrNp.of(A)
    X = _np(X, np.float64)
    rows = _np(rows, np.int64)
    k = X.shape[1]
    Cn = None if C is None else _np(C, np.float64)
    k_out = k if Cn is None else Cn.shape[1]
    Ys = np.zeros((len(rows), k_out)) if Y_sel is None else _np(Y_sel, np.float64).copy()
    r = _load().oracle_spmm_rows(_ptr(rows), len(rows), _ptr(A.row_ptr), _ptr(A.col), _ptr(A.val),
                                 k, _ptr(X), k, _ptr(Cn), k_out, float(alpha), float(beta), _ptr(Ys))
    if r:
        raise ValueError("oracle_spmm_rows: bad arguments")
    return Ys


def gram(X, Y):
    """O2: G = X^T Y, long-double accumulation (bk_oracle.c oracle_gram)."""
    X = _np(X, np.float64); Y = _np(Y, np.float64)
    n, ka = X.shape
    kb = Y.shape[1]
    G = np.zeros((ka, kb))
    _load().oracle_gram(n, ka, kb, _ptr(X), ka, _ptr(Y), kb, _ptr(G))
    return G


def update(X, P, C, a=1.0, s=1.0):
    """O3: returns a X + s P C (bk_oracle.c oracle_update)."""
    X = _np(X, np.float64).copy(); P = _np(P, np.float64); C = _np(C, np.float64)
    n, k = X.shape
    kp = P.shape[1]
    _load().oracle_update(n, kp, k, float(a), _ptr(X), k, float(s), _ptr(P), kp, _ptr(C))
    return X


# --------------------------------------------------------------------------- k x k steps
class Breakdown(Exception):
    def __init__(self, column):
        super().__init__(f"breakdown at column {column}")
        self.column = column


def chol_upper(G, tol):
    """R upper with G = R^T R; breakdown if a pivot <= tol * max|diag(G)| (R6)."""
    G = np.array(G, dtype=np.float64)
    k = G.shape[0]
    scale = max(np.max(np.abs(np.diag(G))), np.finfo(float).tiny)
    R = np.zeros_like(G)
    for j in range(k):
        d = G[j, j] - np.dot(R[:j, j], R[:j, j])
        if not (d > tol * scale):
            raise Breakdown(j)
        R[j, j] = np.sqrt(d)
        for c in range(j + 1, k):
            R[j, c] = (G[j, c] - np.dot(R[:j, j], R[:j, c])) / R[j, j]
    return R


def spd_solve(G, Rhs, tol):
    """Solve G Z = Rhs by Cholesky (O4: (P^T Q) alpha = R^T R)."""
    R = chol_upper(G, tol)
    W = np.linalg.solve(R.T, Rhs)      # forward (lower) solve
    return np.linalg.solve(R, W)       # back (upper) solve


def lu_solve(G, Rhs, tol):
    """Solve G Z = Rhs by LU with partial pivoting (O6); breakdown on a tiny pivot."""
    G = np.array(G, dtype=np.float64)
    k = G.shape[0]
    scale = max(np.max(np.abs(G)), np.finfo(float).tiny)
    A = G.copy(); B = np.array(Rhs, dtype=np.float64).copy()
    for j in range(k):
        p = j + int(np.argmax(np.abs(A[j:, j])))
        if not (abs(A[p, j]) > tol * scale):
            raise Breakdown(j)
        if p != j:
            A[[j, p]] = A[[p, j]]; B[[j, p]] = B[[p, j]]
        for r in range(j + 1, k):
            f = A[r, j] / A[j, j]
            A[r, j:] -= f * A[j, j:]
            B[r] -= f * B[j]
    Z = np.zeros_like(B)
    for j in range(k - 1, -1, -1):
        Z[j] = (B[j] - A[j, j + 1:] @ Z[j + 1:]) / A[j, j]
    return Z


# --------------------------------------------------------------------------- solvers
class Report:
    def __init__(self):
        self.status = "ok"
        self.iterations = 0
        self.converged = False
        self.relres = None
        self.true_relres = None
        self.breakdown_column = -1
        self.history = []


def _colnorms(R):
    return np.sqrt(np.maximum(np.diag(gram(R, R)), 0.0))


def _apply_prec(minv, R):
    if minv is None:
        return R
    if callable(minv):
        return minv(R)
    return R * minv[:, None]


# --------------------------------------------------------------------------- O9 (NEXT-4)
def jacobi_gershgorin(A):
    """O9a: Gershgorin upper bound of the spectrum of D^{-1} A (D = diag A):
    every eigenvalue lies in a disc centred at 1 with radius sum_{j != i} |a_ij| / |a_ii|,
    so lambda_max <= max_i sum_j |a_ij| / |a_ii| (R28)."""
    A = CsrNp.of(A)
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    absum = np.bincount(rows, weights=np.abs(A.val), minlength=A.n_rows)
    return float(np.max(absum / np.abs(A.diag())))


def chebyshev_bounds(A, lmin=None, lmax=None, ratio=30.0):
    """Interval [lmin, lmax] of the Chebyshev preconditioner (R28): lmax defaults to
    the Gershgorin bound O9a, lmin to lmax / ratio."""
    lmax = jacobi_gershgorin(A) if lmax is None or lmax <= 0 else float(lmax)
    lmin = lmax / ratio if lmin is None or lmin <= 0 else float(lmin)
    return lmin, lmax


def chebyshev_prec(A, R, steps, lmin, lmax):
    """O9: Z = p(D^{-1}A) D^{-1} R -- `steps` steps of Chebyshev acceleration for A Z = R from
    Z = 0 with the Jacobi splitting on the interval [lmin, lmax] (Saad, Iterative Methods for
    Sparse Linear Systems, Alg. 12.1, in its order and notation, the
    polynomial stand-in for the paper's AMG preconditioner of Block-CG / Block-BiCGStab,
    PAPER.md P:774):
        theta = (lmax + lmin)/2, delta = (lmax - lmin)/2, sigma = theta/delta, rho_0 = 1/sigma,
        d_0 = D^{-1} R / theta, Z_1 = d_0;
        for j = 1 .. steps-1:  rho_j = 1/(2 sigma - rho_{j-1});
            d_j = rho_j rho_{j-1} d_{j-1} + (2 rho_j / delta) D^{-1} (R - A Z_j);  Z_{j+1} = Z_j + d_j.
    p has degree steps - 1; p(lam) = (1 - T_s((theta - lam)/delta) / T_s(sigma)) / lam."""
    A = CsrNp.of(A)
    R = _np(R, np.float64)
    dinv = 1.0 / A.diag()
    theta = (lmax + lmin) / 2.0
    delta = (lmax - lmin) / 2.0
    sigma = theta / delta
    rho = 1.0 / sigma
    d = dinv[:, None] * R / theta
    Z = d.copy()
    for _ in range(steps - 1):
        rho_n = 1.0 / (2.0 * sigma - rho)
        res = R - spmm(A, Z)
        d = rho_n * rho * d + (2.0 * rho_n / delta) * (dinv[:, None] * res)
        Z = Z + d
        rho = rho_n
    return Z


def block_cg(A, B, X0=None, *, rtol=1e-10, max_iters=1000, precond="none",
             breakdown_tol=1e-13, conv_mode="all", cheb_steps=4, cheb_lmin=None, cheb_lmax=None):
    """O4: block CG (O'Leary 1980, cited PAPER.md P:43; DUNE Block-CG P:1054-1056).

    R = B - A X; Z = M^{-1} R; P = Z; RZ = R^T Z.  Loop: Q = A P;
    (P^T Q) alpha = RZ (Cholesky); X += P alpha; R -= Q alpha; stop when every
    column ||R_c|| <= rtol ||R0_c|| ("defect reduction ... for all
    right-hand-sides"; R5); Z = M^{-1} R; RZn = R^T Z;
    RZ beta = RZn (Cholesky); P = Z + P beta; RZ = RZn.
    M^{-1}: none, Jacobi (D^{-1}) or the Chebyshev polynomial O9 (symmetric positive definite
    for SPD A when lmax bounds the spectrum of D^{-1}A, R28).
    """
    A = CsrNp.of(A)
    B = _np(B, np.float64)
    n, k = B.shape
    X = np.zeros_like(B) if X0 is None else _np(X0, np.float64).copy()
    if precond == "chebyshev":
        lmin, lmax = chebyshev_bounds(A, cheb_lmin, cheb_lmax)
        minv = lambda R: chebyshev_prec(A, R, cheb_steps, lmin, lmax)  # noqa: E731
    else:
        minv = None if precond == "none" else 1.0 / A.diag()
    rep = Report()
    R = B - spmm(A, X)
    r0 = _colnorms(R)
    Z = _apply_prec(minv, R)
    P = Z.copy()
    RZ = gram(R, Z)
    it = 0
    while it < max_iters:
        Q = spmm(A, P)
        PQ = gram(P, Q)
        try:
            alpha = spd_solve(PQ, RZ, breakdown_tol)
        except Breakdown as e:
            rep.status, rep.breakdown_column = "breakdown", e.column
            break
        X = update(X, P, alpha, 1.0, 1.0)
        R = update(R, Q, alpha, 1.0, -1.0)
        it += 1
        nr = _colnorms(R)
        rel = nr / np.where(r0 > 0, r0, 1.0)
        rep.history.append(rel)
        if _converged(rel, conv_mode, rtol):
            rep.converged = True
            break
        Z = _apply_prec(minv, R)
        RZn = gram(R, Z)
        try:
            beta = spd_solve(RZ, RZn, breakdown_tol)
        except Breakdown as e:
            rep.status, rep.breakdown_column = "breakdown", e.column
            break
        P = update(Z, P, beta, 1.0, 1.0)
        RZ = RZn
    return _finish(A, B, X, r0, it, rep)


def block_cg1(A, B, X0=None, *, rtol=1e-10, max_iters=1000, breakdown_tol=1e-13, conv_mode="all"):
    """O11: single-reduction block CG -- O'Leary's block CG (O4) in the one-synchronisation
    form of Chronopoulos & Gear (the communication-avoiding block
    Krylov the paper motivates with, "rediscovered to mitigate the communication
    overhead"; R32).  Every k x k quantity of an iteration comes from ONE reduction
    pass over [R, W = A R]:

        R = B - A X;  W = A R;  G = R^T R;  D = R^T W;  S = D;  S alpha = G (Cholesky);
        P = R;  Q = W.
        Loop:  X += P alpha;  R -= Q alpha;
               W = A R;  Gn = R^T R;  D = R^T W                        (the one reduction)
               stop when every column sqrt(Gn_cc) <= rtol ||R0_c||     (R5)
               G beta = Gn (Cholesky);  S = D - beta^T S beta;  S alpha = Gn (Cholesky);
               P = R + P beta;  Q = W + Q beta;  G = Gn.

    S = P^T A P follows from block-CG orthogonality (R_new^T R_old = 0, Q = A P): with
    P_new = R + P beta, P^T A R = -S beta, so P_new^T A P_new = D - beta^T S beta.  In exact
    arithmetic the iterates are those of O4 (pinned against O4, scalar CG and dense LU in
    tests/test_oracle_pins.py); Q = A P is carried by the recurrence instead of an apply.
    Unpreconditioned.
    """
    A = CsrNp.of(A)
    B = _np(B, np.float64)
    X = np.zeros_like(B) if X0 is None else _np(X0, np.float64).copy()
    rep = Report()
    R = B - spmm(A, X)
    W = spmm(A, R)
    G = gram(R, R)
    D = gram(R, W)
    r0 = np.sqrt(np.maximum(np.diag(G), 0.0))
    S = D
    it = 0
    try:
        alpha = spd_solve(S, G, breakdown_tol)
    except Breakdown as e:
        rep.status, rep.breakdown_column = "breakdown", e.column
        return _finish(A, B, X, r0, it, rep)
    P = R.copy()
    Q = W.copy()
    while it < max_iters:
        X = update(X, P, alpha, 1.0, 1.0)
        R = update(R, Q, alpha, 1.0, -1.0)
        it += 1
        W = spmm(A, R)
        Gn = gram(R, R)
        D = gram(R, W)
        rel = np.sqrt(np.maximum(np.diag(Gn), 0.0)) / np.where(r0 > 0, r0, 1.0)
        rep.history.append(rel)
        if _converged(rel, conv_mode, rtol):
            rep.converged = True
            break
        try:
            beta = spd_solve(G, Gn, breakdown_tol)
            S = D - beta.T @ S @ beta
            alpha = spd_solve(S, Gn, breakdown_tol)
        except Breakdown as e:
            rep.status, rep.breakdown_column = "breakdown", e.column
            break
        P = update(R, P, beta, 1.0, 1.0)
        Q = update(W, Q, beta, 1.0, 1.0)
        G = Gn
    return _finish(A, B, X, r0, it, rep)


def _converged(rel, mode, rtol):
    if mode == "first":
        return rel[0] <= rtol
    return bool(np.all(rel <= rtol))


def _finish(A, B, X, r0, it, rep):
    rep.iterations = it
    rep.relres = rep.history[-1] if rep.history else np.zeros(B.shape[1])
    Rt = B - spmm(A, X)
    rep.true_relres = _colnorms(Rt) / np.where(r0 > 0, r0, 1.0)
    if rep.status == "ok" and not rep.converged:
        rep.status = "not_converged"
    return X, rep


def block_bicgstab(A, B, X0=None, *, rtol=1e-10, max_iters=1000, breakdown_tol=1e-13,
                   conv_mode="all"):
    """O6: block BiCGStab (Guennouni-Jbilou-Sadok form; DUNE Block-BiCGStab P:932-934).

    R = B - A X; Rt = R0; P = R.  Loop: V = A P; (Rt^T V) alpha = Rt^T R (LU);
    S = R - V alpha; T = A S; omega = <T,S>_F / <T,T>_F; X += P alpha + omega S;
    R = S - omega T; test; (Rt^T V) beta = -Rt^T T; P = R + (P - omega V) beta.
    """
    A = CsrNp.of(A)
    B = _np(B, np.float64)
    X = np.zeros_like(B) if X0 is None else _np(X0, np.float64).copy()
    rep = Report()
    R = B - spmm(A, X)
    r0 = _colnorms(R)
    Rt = R.copy()
    P = R.copy()
    it = 0
    while it < max_iters:
        V = spmm(A, P)
        M1 = gram(Rt, V)
        try:
            alpha = lu_solve(M1, gram(Rt, R), breakdown_tol)
        except Breakdown as e:
            rep.status, rep.breakdown_column = "breakdown", e.column
            break
        S = update(R, V, alpha, 1.0, -1.0)
        T = spmm(A, S)
        tt = float(np.trace(gram(T, T)))
        ts = float(np.trace(gram(T, S)))
        if not (tt > 0.0):
            rep.status, rep.breakdown_column = "breakdown", 0
            break
        omega = ts / tt
        X = update(X, P, alpha, 1.0, 1.0) + omega * S
        R = S - omega * T
        it += 1
        rel = _colnorms(R) / np.where(r0 > 0, r0, 1.0)
        rep.history.append(rel)
        if _converged(rel, conv_mode, rtol):
            rep.converged = True
            break
        try:
            beta = lu_solve(M1, -gram(Rt, T), breakdown_tol)
        except Breakdown as e:
            rep.status, rep.breakdown_column = "breakdown", e.column
            break
        P = update(R, P - omega * V, beta, 1.0, 1.0)
    return _finish(A, B, X, r0, it, rep)


def cholqr2(W, tol):
    """CholQR applied twice: W = Q S, S = R2 R1 upper (O5)."""
    R1 = chol_upper(gram(W, W), tol)
    Q1 = W @ np.linalg.inv(R1)
    R2 = chol_upper(gram(Q1, Q1), tol)
    Q = Q1 @ np.linalg.inv(R2)
    return Q, R2 @ R1


def block_gmres(A, B, X0=None, *, rtol=1e-10, max_iters=1000, restart=30,
                breakdown_tol=1e-13, conv_mode="all"):
    """O5: block GMRES(m) with block classical Gram-Schmidt twice (BCGS2) and CholQR2.

    R0 = B - A X; [V_0, S] = CholQR2(R0).  For j = 0..m-1: W = A V_j; two
    passes of {Hp = [V_0..V_j]^T W; W -= [V_0..V_j] Hp}, H[:, j] = H1 + H2;
    [V_{j+1}, H_{j+1,j}] = CholQR2(W).  Per-column residual norms are those of
    the least-squares problem min ||E_1 S - Hbar Y|| (solved here by lstsq,
    the plain definition).  At the end of a cycle X += [V_0..V_j] Y, restart.
    """
    A = CsrNp.of(A)
    B = _np(B, np.float64)
    n, k = B.shape
    X = np.zeros_like(B) if X0 is None else _np(X0, np.float64).copy()
    rep = Report()
    R = B - spmm(A, X)
    r0 = _colnorms(R)
    it = 0
    m = restart
    done = False
    while not done and it < max_iters:
        try:
            V0, S = cholqr2(R, breakdown_tol)
        except Breakdown as e:
            rep.status, rep.breakdown_column = "breakdown", e.column
            break
        Vs = [V0]
        H = np.zeros(((m + 1) * k, m * k))
        g = np.zeros(((m + 1) * k, k)); g[:k] = S
        Ysol = None
        jlast = -1
        for j in range(m):
            W = spmm(A, Vs[j])
            Vcat = np.concatenate(Vs, axis=1)
            Hc = np.zeros(((j + 1) * k, k))
            for _ in range(2):
                Hp = gram(Vcat, W)
                W = W - Vcat @ Hp
                Hc += Hp
            H[:(j + 1) * k, j * k:(j + 1) * k] = Hc
            try:
                Vn, Hn = cholqr2(W, breakdown_tol)
            except Breakdown as e:
                rep.status, rep.breakdown_column = "breakdown", e.column
                done = True
                break
            H[(j + 1) * k:(j + 2) * k, j * k:(j + 1) * k] = Hn
            Vs.append(Vn)
            it += 1
            Hb = H[:(j + 2) * k, :(j + 1) * k]
            gb = g[:(j + 2) * k]
            Ysol = np.linalg.lstsq(Hb, gb, rcond=None)[0]
            res = gb - Hb @ Ysol
            rel = np.sqrt((res * res).sum(axis=0)) / np.where(r0 > 0, r0, 1.0)
            rep.history.append(rel)
            jlast = j
            if _converged(rel, conv_mode, rtol):
                rep.converged = True
                done = True
                break
            if it >= max_iters:
                done = True
                break
        if jlast >= 0 and Ysol is not None:
            Vcat = np.concatenate(Vs[:jlast + 1], axis=1)
            X = X + Vcat @ Ysol
        if not done:
            R = B - spmm(A, X)
    return _finish(A, B, X, r0, it, rep)


def dense_solve(A, B):
    """O7: dense reference X = A^{-1} B by LU with partial pivoting (numpy/LAPACK), tiny N."""
    D = np.zeros((A.n_rows, A.n_cols))
    A = CsrNp.of(A)
    for i in range(A.n_rows):
        for p in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[p]] += A.val[p]
    return np.linalg.solve(D, _np(B, np.float64))


SOLVERS = {"cg": block_cg, "gmres": block_gmres, "bicgstab": block_bicgstab, "cg1": block_cg1}


# ---------------------------------------------------------------------------
# O8: the DIRK window as one matrix equation.
# M = mass * I (finite volumes), K: CSR stiffness, A: Butcher matrix of a
# stiffly accurate DIRK method (m x m, row-major), s time steps per window,
# k = s m columns.  All dense / tiny N.
# ---------------------------------------------------------------------------
def _dense(A):
    A = CsrNp.of(A)
    D = np.zeros((A.n_rows, A.n_cols))
    for i in range(A.n_rows):
        for p in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[p]] += A.val[p]
    return D


def dirk_sequential(K, mass, A_tab, Bcols, y_n, tau, s):
    """Classical stepping of eq. (stiffly-accurate-DIRK): for step q and stage i
    (1/tau) M (y^(q,i) - y^q) + sum_{j<=i} a_ij K y^(q,j) = sum_{j<=i} a_ij b(t^(q,j)),
    y^{q+1} = y^(q,m) (stiffly accurate).  Bcols[:, q m + j] = b(t^(q,j)).
    Returns Y (N x s m), column q m + i = y^(q,i).  Dense solves (tiny N)."""
    Kd = _dense(K)
    N = Kd.shape[0]
    A = np.asarray(A_tab, dtype=np.float64)
    m = A.shape[0]
    Bc = _np(Bcols, np.float64)
    Y = np.zeros((N, s * m))
    yq = _np(y_n, np.float64).reshape(N).copy()
    for q in range(s):
        for i in range(m):
            lhs = mass / tau * np.eye(N) + A[i, i] * Kd
            rhs = mass / tau * yq
            for j in range(i + 1):
                rhs = rhs + A[i, j] * Bc[:, q * m + j]
            for j in range(i):
                rhs = rhs - A[i, j] * (Kd @ Y[:, q * m + j])
            Y[:, q * m + i] = np.linalg.solve(lhs, rhs)
        yq = Y[:, q * m + m - 1].copy()
    return Y


def theta_stepping(K, mass, theta, b, y0, tau, s):
    """Closed-form Theta scheme, Example ex:time-stepping-matrices:
    (M/tau + Theta K) y^{q+1} = Theta b^{q+1} + M y^q / tau + (1 - Theta)(b^q - K y^q), q = 0..s-1,
    M = mass I; b[:, q] = b(t^q) for q = 0..s.  Returns Y (N x s), column q = y^{q+1}.  Dense solves."""
    Kd = _dense(K)
    N = Kd.shape[0]
    b = _np(b, np.float64)
    y = _np(y0, np.float64).reshape(N).copy()
    Y = np.zeros((N, s))
    for q in range(s):
        y = np.linalg.solve(mass / tau * np.eye(N) + theta * Kd,
                            theta * b[:, q + 1] + mass / tau * y + (1.0 - theta) * (b[:, q] - Kd @ y))
        Y[:, q] = y
    return Y


def dirk_all_at_once(K, mass, A1, A2, B, B0):
    """Eq. (general-system-time-steps), P:104-126 with the window matrices of P:260-288:
    [A1 (x) M + A2 (x) K] vec(Y) = [A2 (x) I_N] vec(B) + vec(B0), vec = column stacking
    (X_1^T, ..., X_k^T)^T; i.e. M Y A1^T + K Y A2^T = B A2^T + B0.  Dense Kronecker solve."""
    Kd = _dense(K)
    N = Kd.shape[0]
    A1 = np.asarray(A1, dtype=np.float64)
    A2 = np.asarray(A2, dtype=np.float64)
    Md = mass * np.eye(N)
    lhs = np.kron(A1, Md) + np.kron(A2, Kd)
    Bm = _np(B, np.float64)
    rhs = np.kron(A2, np.eye(N)) @ Bm.T.reshape(-1) + _np(B0, np.float64).T.reshape(-1)
    return np.linalg.solve(lhs, rhs).reshape(A1.shape[0], N).T


def dirk_fixed_point(L, K, mass, tau, A1, A2, B, B0, Y0, iters, inner=None):
    """Splitting fixed point, eq. (matrix-splitting) and (matrix-fixed-point-equation), P:357-395:
    beta = A2[0,0]; (M/tau + beta K) Y^j = -M Y^{j-1} (A1 - I/tau)^T - K Y^{j-1} (A2 - beta I)^T
                                           + B A2^T + B0,   j = 1..iters.
    L = M/tau + beta K (CSR).  inner: None = exact (dense) solves, else a callable
    inner(L, Rhs, X0) -> Y (e.g. a block Krylov oracle).  Returns (Y, [Y^1, ..., Y^iters])."""
    A1 = np.asarray(A1, dtype=np.float64)
    A2 = np.asarray(A2, dtype=np.float64)
    k = A1.shape[0]
    beta = A2[0, 0]
    Y = _np(Y0, np.float64).copy()
    Bm = _np(B, np.float64)
    fixed = Bm @ A2.T + _np(B0, np.float64)
    Ld = _dense(L) if inner is None else None
    hist = []
    for _ in range(iters):
        rhs = (-mass * Y @ (A1 - np.eye(k) / tau).T
               - spmm(K, Y) @ (A2 - beta * np.eye(k)).T + fixed)
        Y = np.linalg.solve(Ld, rhs) if inner is None else inner(L, rhs, Y)
        hist.append(Y.copy())
    return Y, hist


# --------------------------------------------------------------------------- O10 (NEXT-3)
from .alg1 import (DRProblem, algorithm1, dr_f, dr_jacobian, iota, residual as alg1_residual,  # noqa: E402,F401
                   sequential_dirk, shift as alg1_shift, window_A)
