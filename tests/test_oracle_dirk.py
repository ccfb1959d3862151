"""Pins of the DIRK window oracle (O8) against what the paper and the
mathematics fix -- not against itself:
  * the all-at-once matrix equation (eq. general-system-time-steps, window matrices
    P:260-288) equals classical sequential SDIRK stepping (eq. stiffly-accurate-DIRK);
  * the eliminated-stage Theta-method window equals the closed-form Theta scheme
    (Example ex:time-stepping-matrices P:302-334);
  * the splitting fixed point (eq. matrix-fixed-point-equation) is exact after k
    outer iterations, column c after c + 1, because the coupling is strictly lower triangular.
"""
import math

import numpy as np
import pytest

import oracle
import synth


def _problem(n=10, tau=0.05, conv=True, seed=0):
    K = synth.convdiff2d(n, tau=float("inf"), gamma=1.0, v=(1.0, 0.5) if conv else (0.0, 0.0))
    mass = (1.0 / n) ** 2
    rng = np.random.default_rng(seed)
    N = n * n
    return K, mass, rng.uniform(-1, 1, N), rng.uniform(-1, 1, N), rng.uniform(-1, 1, N)


def _window(A_tab, s, tau, f, g, y0, mass):
    """B columns b(t^(q,i)) = sin(1 + t) f + g + e_(q,i) (independent seeded components, so the
    block right-hand side has full column rank), B0 = (1/tau) M y^n in the first m columns."""
    m = len(A_tab)
    c = np.array(A_tab).sum(1)
    e = np.random.default_rng(7).uniform(-0.5, 0.5, (len(f), s * m))
    B = np.stack([math.sin(1.0 + (q + c[i]) * tau) * f + g + e[:, q * m + i] for q in range(s) for i in range(m)], 1)
    B0 = np.zeros((len(f), s * m))
    B0[:, :m] = (mass / tau * y0)[:, None]
    return B, B0


@pytest.mark.parametrize("tab,s", [("sdirk2", 2), ("sdirk2", 4), ("sdirk3", 2)])
def test_all_at_once_equals_sequential_sdirk(tab, s):
    tau = 0.05
    K, mass, f, g, y0 = _problem(tau=tau)
    A_tab = synth.SDIRK2 if tab == "sdirk2" else synth.SDIRK3
    A1, A2 = synth.window_matrices(A_tab, s, tau)
    B, B0 = _window(A_tab, s, tau, f, g, y0, mass)
    Ys = oracle.dirk_sequential(K, mass, A_tab, B, y0, tau, s)
    Ya = oracle.dirk_all_at_once(K, mass, A1.numpy(), A2.numpy(), B, B0)
    assert np.abs(Ys - Ya).max() <= 1e-12 * np.abs(Ya).max()


def test_theta_window_equals_closed_form_theta_scheme():
    """Eliminated explicit stage: window of s Crank-Nicolson steps vs
    (M/tau + theta K) y^{n+1} = theta b^{n+1} + M y^n / tau + (1 - theta)(b^n - K y^n)."""
    tau, theta, s = 0.05, 0.5, 3
    K, mass, f, g, y0 = _problem(tau=tau)
    Kd = oracle._dense(K)
    N = Kd.shape[0]
    b = [math.sin(1.0 + q * tau) * f + g for q in range(s + 1)]          # b(t^n), ..., b(t^{n+s})
    A1, A2 = synth.window_matrices([[theta]], s, tau, a_elim=[1.0 - theta])
    B = np.stack(b[1:], 1)
    B0 = np.zeros((N, s))
    B0[:, 0] = mass / tau * y0 - (1.0 - theta) * (Kd @ y0 - b[0])         # Example P:329-333
    Ya = oracle.dirk_all_at_once(K, mass, A1.numpy(), A2.numpy(), B, B0)
    y = y0.copy()
    for q in range(s):
        y = np.linalg.solve(mass / tau * np.eye(N) + theta * Kd,
                            theta * b[q + 1] + mass / tau * y + (1.0 - theta) * (b[q] - Kd @ y))
        assert np.abs(Ya[:, q] - y).max() <= 1e-12 * np.abs(y).max()
    # oracle.theta_stepping is that recurrence (used by the library window tests)
    Yt = oracle.theta_stepping(K, mass, theta, np.stack(b, 1), y0, tau, s)
    assert np.abs(Ya - Yt).max() <= 1e-12 * np.abs(Yt).max()


@pytest.mark.parametrize("tab,s", [("sdirk2", 2), ("sdirk3", 2)])
def test_fixed_point_exact_after_k_iterations(tab, s):
    tau = 0.05
    K, mass, f, g, y0 = _problem(tau=tau)
    A_tab = synth.SDIRK2 if tab == "sdirk2" else synth.SDIRK3
    gamma = A_tab[0][0]
    L = synth.convdiff2d(10, tau=tau, gamma=gamma)                       # M/tau + beta K, beta = A2[0,0]
    A1, A2 = synth.window_matrices(A_tab, s, tau)
    k = A1.shape[0]
    B, B0 = _window(A_tab, s, tau, f, g, y0, mass)
    Ya = oracle.dirk_all_at_once(K, mass, A1.numpy(), A2.numpy(), B, B0)
    _, hist = oracle.dirk_fixed_point(L, K, mass, tau, A1.numpy(), A2.numpy(), B, B0, np.zeros_like(B), k)
    scale = np.abs(Ya).max()
    for j, Yj in enumerate(hist):                                        # after j + 1 iterations
        err = np.abs(Yj - Ya).max(axis=0) / scale
        assert np.all(err[:j + 1] <= 1e-12), (j, err)                    # columns 0..j exact
    assert np.abs(hist[k - 2][:, k - 1] - Ya[:, k - 1]).max() > 1e-6 * scale   # not before


def test_fixed_point_with_block_krylov_inner_solves():
    """Inner solves by the block GMRES oracle to 1e-12: the window solution within ~kappa * rtol."""
    tau, s = 0.05, 2
    K, mass, f, g, y0 = _problem(tau=tau)
    A1, A2 = synth.window_matrices(synth.SDIRK2, s, tau)
    L = synth.convdiff2d(10, tau=tau, gamma=synth.SDIRK2_GAMMA)
    B, B0 = _window(synth.SDIRK2, s, tau, f, g, y0, mass)
    Ya = oracle.dirk_all_at_once(K, mass, A1.numpy(), A2.numpy(), B, B0)

    def inner(Lm, rhs, X0):
        X, rep = oracle.block_gmres(Lm, rhs, None, rtol=1e-12, restart=200, max_iters=400)
        assert rep.converged
        return X
    Y, _ = oracle.dirk_fixed_point(L, K, mass, tau, A1.numpy(), A2.numpy(), B, B0, np.zeros_like(B), 4, inner)
    assert np.linalg.norm(Y - Ya) <= 1e-9 * np.linalg.norm(Ya)
