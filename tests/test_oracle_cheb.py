"""Pins of the Chebyshev polynomial preconditioner oracle (O9, the
polynomial stand-in for the paper's AMG preconditioner) against what the
mathematics fixes -- not against itself:
  * the recurrence equals the closed form p(D^-1 A) D^-1 R with
    p(lam) = (1 - T_s((theta - lam)/delta) / T_s(sigma)) / lam, evaluated in the eigenbasis of
    D^-1/2 A D^-1/2 with numpy's Chebyshev basis (R28);
  * one step is scaled Jacobi, D^-1 R / theta;
  * the Gershgorin bound O9a bounds the spectrum of D^-1 A from above (dense eigenvalues) and is
    attained-in-the-limit for the Dirichlet Laplacian (2);
  * block PCG with it converges to the dense-LU solution in fewer iterations than plain CG, and
    its preconditioner is symmetric positive definite.
"""
import numpy as np
import pytest

import oracle
import synth


def _dense(A):
    return oracle._dense(A)


def _spd_matrix():
    return synth.richards3d(6, 5, 4)          # exactly symmetric SPD, heterogeneous coefficients


def _closed_form(Ad, R, steps, lmin, lmax):
    d = np.diag(Ad)
    s = 1.0 / np.sqrt(d)
    Ah = s[:, None] * Ad * s[None, :]
    lam, V = np.linalg.eigh(Ah)
    theta, delta = (lmax + lmin) / 2, (lmax - lmin) / 2
    T = np.polynomial.chebyshev.Chebyshev.basis(steps)
    p = (1.0 - T((theta - lam) / delta) / T(theta / delta)) / lam
    return s[:, None] * (V @ (p[:, None] * (V.T @ (s[:, None] * R))))


@pytest.mark.parametrize("steps", [1, 2, 3, 5, 8])
def test_recurrence_equals_closed_form(steps):
    A = _spd_matrix()
    Ad = _dense(A)
    R = synth.multivector(A.n_rows, 3, 2).numpy()
    lmin, lmax = oracle.chebyshev_bounds(A)
    Z = oracle.chebyshev_prec(A, R, steps, lmin, lmax)
    Zc = _closed_form(Ad, R, steps, lmin, lmax)
    assert np.abs(Z - Zc).max() <= 1e-11 * np.abs(Zc).max()


def test_one_step_is_scaled_jacobi():
    A = _spd_matrix()
    R = synth.multivector(A.n_rows, 4, 3).numpy()
    Z = oracle.chebyshev_prec(A, R, 1, 0.1, 1.9)
    assert np.array_equal(Z, (1.0 / np.diag(_dense(A)))[:, None] * R / 1.0)


def test_gershgorin_bounds_the_spectrum():
    for A in (_spd_matrix(), synth.convdiff2d(8), synth.diffreact3d(5)):
        Ad = _dense(A)
        lam = np.linalg.eigvals(Ad / np.diag(Ad)[:, None])
        g = oracle.jacobi_gershgorin(A)
        assert lam.real.max() <= g * (1 + 1e-14)
    # 1-D Dirichlet Laplacian tridiag(-1, 2, -1): bound 2, lambda_max = 1 + cos(pi/(n+1)) -> 2
    n = 50
    rp = np.concatenate([[0], np.cumsum([2] + [3] * (n - 2) + [2])]).astype(np.int32)
    cols, vals = [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                cols.append(j)
                vals.append(2.0 if i == j else -1.0)
    L = oracle.CsrNp(n, n, rp, np.array(cols, np.int32), np.array(vals))
    assert oracle.jacobi_gershgorin(L) == 2.0
    assert 2.0 - (1.0 + np.cos(np.pi / (n + 1))) < 2e-3


def test_preconditioner_is_spd():
    A = _spd_matrix()
    N = A.n_rows
    lmin, lmax = oracle.chebyshev_bounds(A)
    I = np.eye(N)
    M = np.concatenate([oracle.chebyshev_prec(A, I[:, c:c + 24], 4, lmin, lmax) for c in range(0, N, 24)], 1)
    assert np.abs(M - M.T).max() <= 1e-12 * np.abs(M).max()
    assert np.linalg.eigvalsh((M + M.T) / 2).min() > 0


@pytest.mark.parametrize("k", [1, 4])
def test_pcg_converges_to_dense_solution_in_fewer_iterations(k):
    A = synth.laplace_mms2d(24)               # Poisson: kappa ~ 230 (the c4/c5 operators at large tau)
    B = synth.multivector(A.n_rows, k, 2).numpy()
    Xd = oracle.dense_solve(A, B)
    X0, rep0 = oracle.block_cg(A, B, rtol=1e-10, max_iters=500)
    X1, rep1 = oracle.block_cg(A, B, rtol=1e-10, max_iters=500, precond="chebyshev", cheb_steps=4)
    assert rep0.converged and rep1.converged
    assert 2 * rep1.iterations < rep0.iterations        # 84 -> 24 (k = 1), 59 -> 21 (k = 4)
    kappa = np.linalg.cond(_dense(A))
    for X in (X0, X1):
        assert np.linalg.norm(X - Xd) <= 10 * kappa * 1e-10 * np.linalg.norm(Xd)
