"""Pins of the Algorithm 1 oracle (O10; §2.2) against
what the paper and the mathematics fix -- not against itself:
  * iota / shift: the paper's formulas on SPEC's examples;
  * f: conservation (the diffusion fluxes cancel in the sum over cells) and the closed form for
    a constant field; Df: central finite differences of f (O(eps^2));
  * the pipelined residual R(Y) vanishes when the window holds the exact stage
    values of a sequential DIRK run solved by scipy's MINPACK root finder (independent solver),
    for windows starting at every stage offset;
  * Algorithm 1 with window 1 (classical Newton per stage) and with windows 2..4 (pipelining)
    reproduces that sequential trajectory.
"""
import numpy as np
import pytest
from scipy import optimize

import oracle
import synth


def _problem(nx=6, ny=5, nz=4, tau=0.05, seed=1):
    y0, g = synth.dr_fields(nx, ny, nz, seed)
    return oracle.DRProblem(nx, ny, nz, y0.numpy(), g.numpy(), tau)


def _root(G, x0):
    r = optimize.root(G, x0, method="hybr", options={"xtol": 1e-13})
    scale = np.abs(G(np.zeros_like(x0))).max() + np.abs(G(x0)).max()
    assert np.abs(G(r.x)).max() <= 1e-13 * scale            # converged to rounding level
    return r.x


def test_iota_and_shift_examples():
    assert oracle.iota(0, 1, 3) == (0, 1)
    assert oracle.iota(0, 4, 3) == (1, 1)
    assert oracle.iota(2, 3, 3) == (2, 3)
    Y = np.arange(12.0).reshape(4, 3)
    assert np.array_equal(oracle.alg1_shift(Y), Y[:, [1, 2, 2]])
    assert np.array_equal(oracle.alg1_shift(Y[:, :1]), Y[:, :1])


def test_f_conservation_and_constant_field():
    P = _problem()
    u = np.random.default_rng(0).uniform(0, 1, P.N)
    t = 0.3
    F = oracle.dr_f(P, t, u)
    h3 = P.h ** 3
    src = h3 * (u - u * u) - h3 * np.sin(1.0 + t) * P.g
    assert abs((F - src).sum()) <= 1e-15 * np.abs(F - src).sum() * P.N
    c = 0.37
    Fc = oracle.dr_f(P, t, np.full(P.N, c))
    assert np.allclose(Fc, h3 * (c - c * c) - h3 * np.sin(1.0 + t) * P.g, rtol=0, atol=1e-18)


def test_jacobian_is_the_derivative_of_f():
    P = _problem()
    rng = np.random.default_rng(1)
    u = rng.uniform(0, 1, P.N)
    J = oracle.dr_jacobian(P, u)
    for _ in range(3):
        v = rng.uniform(-1, 1, P.N)
        e = 1e-5
        fd = (oracle.dr_f(P, 0.0, u + e * v) - oracle.dr_f(P, 0.0, u - e * v)) / (2 * e)
        Jv = oracle.spmm(J, v[:, None])[:, 0]
        assert np.abs(Jv - fd).max() <= 1e-8 * np.abs(Jv).max()
    Js = oracle.dr_jacobian(P, u, shift=2.5, scale=0.5)
    assert np.allclose(oracle._dense(Js), 2.5 * np.eye(P.N) + 0.5 * oracle._dense(J), rtol=0, atol=1e-15)


@pytest.mark.parametrize("tab", ["sdirk2", "sdirk3"])
def test_residual_vanishes_on_the_sequential_solution(tab):
    P = _problem()
    A = synth.SDIRK2 if tab == "sdirk2" else synth.SDIRK3
    m = len(A)
    nst = 3
    stages = []
    traj = oracle.sequential_dirk(P, A, nst, _root, stages)
    S = np.stack(stages, 1)                                   # all stage values, global order
    scale = np.abs(P.mass / P.tau * S).max()
    for w in (1, 2, m, m + 2):
        for g0 in range(0, nst * m - w + 1):
            n = g0 // m
            yn = P.y0 if n == 0 else traj[:, n - 1]
            c = np.asarray(A).sum(1)
            fh = [oracle.dr_f(P, n * P.tau + P.tau * c[j], S[:, n * m + j]) for j in range(g0 % m)]
            R, _ = oracle.alg1_residual(P, A, S[:, g0:g0 + w], g0, yn, fh)
            assert np.abs(R).max() <= 1e-12 * scale, (w, g0, np.abs(R).max() / scale)


@pytest.mark.parametrize("tab,window", [("sdirk2", 1), ("sdirk2", 2), ("sdirk2", 4), ("sdirk3", 1), ("sdirk3", 3)])
def test_algorithm1_reproduces_sequential_trajectory(tab, window):
    P = _problem()
    A = synth.SDIRK2 if tab == "sdirk2" else synth.SDIRK3
    nst = 4
    ref = oracle.sequential_dirk(P, A, nst, _root)
    traj, its = oracle.algorithm1(P, A, nst, window, eps=1e-13 * np.sqrt(P.N) * P.mass / P.tau)
    assert traj.shape == ref.shape
    assert np.abs(traj - ref).max() <= 1e-10 * np.abs(ref).max()
    assert len(its) == nst * len(A)
    if window == 1:
        assert max(its) <= 6                                  # Newton with the exact Jacobian
