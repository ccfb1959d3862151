"""O10: Algorithm 1 "Block Krylov Time Stepping with Pipelining"
(§2.2) on the nonlinear diffusion-reaction problem.  TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py); independent of the CUDA path.

Problem (R29; the c3 operator family, R16): M y' + f(t, y) = 0 on an nx x ny x nz
cell-centred lattice, h = 1/nx, Neumann boundary, M = h^3 I,
    f(t,u)_a = sum_{b in nb(a)} h D_ab (u_a - u_b) + h^3 (u_a - u_a^2) - h^3 sin(1 + t) g_a,
    D_ab = 1 + (u_a^2 + u_b^2)/2,
and its Jacobian Df(u) (J_aa = sum_b h (D_ab + u_a (u_a - u_b)) + h^3 (1 - 2 u_a),
J_ab = h (u_b (u_a - u_b) - D_ab)).

Time stepping: a stiffly accurate DIRK tableau A (m stages, c = A 1), t^n = n tau.  The
pipelined window holds w consecutive global stages g0 .. g0+w-1 (stage s belongs to step
s // m, stage index s % m; the paper's iota(n, k) of P:574-580 with 1-based k).  With the
window matrices of eq. (time-stepping-matrices-multiple-parallel-time-steps) restricted to
rows/columns g0 .. g0+w-1 (the paper's A_1^{(n,k)}, A_2^{(n,k)}, "submatrices ... starting at
the index (k,k)") the residual is (sign reading R30)
    R(Y) = M Y A1^T + F(T, Y) A2^T - B0,
    B0_i = (1/tau) M y^n - sum_{accepted j < c_i} a_{c_i j} f(t^n + tau c_j, y^{(n,j)})
           if column i belongs to the current step n, else 0.
Algorithm 1: Y = (y0, ..., y0); per stage: Y <- shift(Y); Newton loop:
R <- R(Y); if ||R_0|| < eps accept column 0 and break; J <- (1/tau) M + a_kk Df(t_0, Y_0);
solve J V = R; Y <- Y - V.
"""
from __future__ import annotations

import numpy as np

from . import CsrNp, spmm


class DRProblem:
    """Nonlinear diffusion-reaction lattice problem (R29)."""

    def __init__(self, nx, ny, nz, y0, g, tau):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.N = self.nx * self.ny * self.nz
        self.h = 1.0 / self.nx
        self.y0 = np.asarray(y0, np.float64).reshape(self.N)
        self.g = np.asarray(g, np.float64).reshape(self.N)
        self.tau = float(tau)
        self.mass = self.h ** 3

    def neighbours(self):
        """[(offset, mask)] of the 6 faces, ascending offset (x fastest)."""
        r = np.arange(self.N)
        ix, iy, iz = r % self.nx, (r // self.nx) % self.ny, r // (self.nx * self.ny)
        s1, s2 = self.nx, self.nx * self.ny
        return [(-s2, iz > 0), (-s1, iy > 0), (-1, ix > 0), (1, ix < self.nx - 1), (s1, iy < self.ny - 1),
                (s2, iz < self.nz - 1)]


def dr_f(P: DRProblem, t, U):
    """f(t, u) column by column (U: N or N x w; t scalar or per column)."""
    U = np.asarray(U, np.float64)
    one = U.ndim == 1
    U2 = U[:, None] if one else U
    tt = np.broadcast_to(np.asarray(t, np.float64), (U2.shape[1],))
    h = P.h
    F = h ** 3 * (U2 - U2 * U2) - h ** 3 * np.sin(1.0 + tt)[None, :] * P.g[:, None]
    idx = np.arange(P.N)
    for off, m in P.neighbours():
        b = np.where(m, idx + off, idx)
        ub = U2[b]
        D = 1.0 + 0.5 * (U2 * U2 + ub * ub)
        F += np.where(m[:, None], h * D * (U2 - ub), 0.0)
    return F[:, 0] if one else F


def dr_jacobian(P: DRProblem, u, shift=0.0, scale=1.0):
    """CSR of shift * I + scale * Df(u) (7-point pattern, ascending columns)."""
    u = np.asarray(u, np.float64)
    h = P.h
    diag = shift + scale * h ** 3 * (1.0 - 2.0 * u)
    idx = np.arange(P.N)
    offs = []
    for off, m in P.neighbours():
        b = np.where(m, idx + off, idx)
        ub = u[b]
        D = 1.0 + 0.5 * (u * u + ub * ub)
        diag = diag + np.where(m, scale * h * (D + u * (u - ub)), 0.0)
        offs.append((off, m, scale * h * (ub * (u - ub) - D)))
    rows, cols, vals = [], [], []
    for off, m, v in offs[:3] + [(0, np.ones(P.N, bool), diag)] + offs[3:]:
        rows.append(idx[m]); cols.append(idx[m] + off); vals.append(v[m])
    rows, cols, vals = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    order = np.lexsort((cols, rows))
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=P.N))]).astype(np.int32)
    return CsrNp(P.N, P.N, rp, cols[order].astype(np.int32), vals[order])


def iota(n, k, m):
    """iota(n, k) = (n + floor((k-1)/m), ((k-1) mod m) + 1) (1-based stage, the
    paper's "k mod m" read as the 1-based wrap-around, R31)."""
    return n + (k - 1) // m, (k - 1) % m + 1


def shift(Y):
    """shift((Y_1, ..., Y_{s-1}, Y_s)) = (Y_2, ..., Y_s, Y_s) (eq. shift)."""
    return np.concatenate([Y[:, 1:], Y[:, -1:]], axis=1)


def window_A(A_tab, tau, g0, w):
    """A1^{(n,k)}, A2^{(n,k)}: rows / columns g0 .. g0+w-1 of the multi-step window matrices
    A2 = I_s (x) A, A1 = (1/tau)(I - E), E[q m + i, q m - 1] = 1 (R24)."""
    A = np.asarray(A_tab, np.float64)
    m = A.shape[0]
    A1 = np.zeros((w, w))
    A2 = np.zeros((w, w))
    for i in range(w):
        si = g0 + i
        qi, ci = divmod(si, m)
        A1[i, i] = 1.0 / tau
        for j in range(w):
            sj = g0 + j
            qj, cj = divmod(sj, m)
            if qj == qi:
                A2[i, j] = A[ci, cj]
            if ci >= 0 and qi >= 1 and sj == qi * m - 1:
                A1[i, j] = -1.0 / tau
    return A1, A2


def residual(P, A_tab, Y, g0, yn, fhist):
    """R(Y) = M Y A1^T + F(T, Y) A2^T - B0 for the window starting at global stage g0;
    yn = y^n of the current step n = g0 // m, fhist[j] = f of its accepted stages j < g0 % m."""
    A = np.asarray(A_tab, np.float64)
    m = A.shape[0]
    c = A.sum(1)
    w = Y.shape[1]
    n = g0 // m
    A1, A2 = window_A(A, P.tau, g0, w)
    T = np.array([((g0 + i) // m) * P.tau + P.tau * c[(g0 + i) % m] for i in range(w)])
    F = dr_f(P, T, Y)
    B0 = np.zeros_like(Y)
    for i in range(w):
        q, ci = divmod(g0 + i, m)
        if q == n:
            B0[:, i] = P.mass / P.tau * yn
            for j, fj in enumerate(fhist):
                B0[:, i] -= A[ci, j] * fj
    return P.mass * Y @ A1.T + F @ A2.T - B0, F


def _solve(J, R):
    D = np.zeros((J.n_rows, J.n_cols))
    for i in range(J.n_rows):
        D[i, J.col[J.row_ptr[i]:J.row_ptr[i + 1]]] = J.val[J.row_ptr[i]:J.row_ptr[i + 1]]
    return np.linalg.solve(D, R)


def algorithm1(P: DRProblem, A_tab, n_steps, window, eps, max_newton=50, solve=None):
    """Algorithm 1.  Returns (trajectory N x n_steps = y^1 .. y^{n_steps},
    newton iterations per accepted stage).  solve(J, R) -> V defaults to a dense LU solve."""
    A = np.asarray(A_tab, np.float64)
    m = A.shape[0]
    c = A.sum(1)
    solve = solve or _solve
    w = int(window)
    Y = np.repeat(P.y0[:, None], w, axis=1)                  # Y^(0,0) = (y0, ..., y0)
    yn = P.y0.copy()
    fhist = []
    traj, its = [], []
    g0 = 0
    first = True
    while g0 < n_steps * m:
        if not first:
            Y = shift(Y)                                      # line 4
        first = False
        for i in range(max_newton + 1):
            R, F = residual(P, A, Y, g0, yn, fhist)
            if np.linalg.norm(R[:, 0]) < eps:                 # lines 6-9
                break
            if i == max_newton:
                raise RuntimeError(f"stage {g0}: Newton did not converge, ||R_0|| = {np.linalg.norm(R[:, 0])}")
            ck = g0 % m
            t0 = (g0 // m) * P.tau + P.tau * c[ck]
            J = dr_jacobian(P, Y[:, 0], shift=P.mass / P.tau, scale=A[ck, ck])   # line 10
            V = solve(J, R)                                   # line 11 "solve JV = R"
            Y = Y - V                                         # line 12
        its.append(i)
        ck = g0 % m
        if ck == m - 1:                                       # stiffly accurate: y^{n+1} = last stage
            yn = Y[:, 0].copy()
            traj.append(yn)
            fhist = []
        else:
            fhist.append(F[:, 0].copy())
        g0 += 1
    return np.stack(traj, 1), its


def sequential_dirk(P: DRProblem, A_tab, n_steps, stage_solve, stages=None):
    """Classical stage-by-stage DIRK (eq. stiffly-accurate-DIRK):
    M (y_s - y^n)/tau + sum_{j <= s} a_sj f(t^n + tau c_j, y_j) = 0, each stage solved by
    stage_solve(G, x0) -> root of G (an independent nonlinear solver in the pins); every stage
    value is appended to `stages` if given."""
    A = np.asarray(A_tab, np.float64)
    m = A.shape[0]
    c = A.sum(1)
    yn = P.y0.copy()
    traj = []
    for n in range(n_steps):
        fs = []
        for s in range(m):
            t = n * P.tau + P.tau * c[s]
            known = sum(A[s, j] * fs[j] for j in range(s)) if s else 0.0

            def G(y, t=t, known=known, s=s):
                return P.mass * (y - yn) / P.tau + known + A[s, s] * dr_f(P, t, y)
            y = stage_solve(G, yn if s == 0 else ys)
            ys = y
            fs.append(dr_f(P, t, y))
            if stages is not None:
                stages.append(y)
        yn = ys
        traj.append(yn)
    return np.stack(traj, 1)
