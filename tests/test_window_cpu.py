"""bk_dirk_window (host-only library entry point, no GPU): the window matrices of NEXT-1 built
from a Butcher tableau, pinned by the paper's worked example and by the all-at-once = sequential
identity (§2.1)."""
import math
import os

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "theta_window.txt")


@pytest.fixture(scope="module")
def bk():
    import paper_2504_02117_b200 as m
    return m


def test_theta_method_window_is_the_papers_example(bk):
    """Example ex:time-stepping-matrices: the Theta-method written as the explicit-first-stage
    tableau [[0, 0], [1 - Theta, Theta]] gives, after elimination, tau A1 = lower
    bidiagonal (1, -1) and A2 = lower bidiagonal (Theta, 1 - Theta) -- the golden file's values."""
    lines = [ln.strip() for ln in open(GOLD) if ln.strip() and not ln.startswith("#")]
    theta = float(lines[0].split()[1]); s = int(lines[1].split()[1]); tau = float(lines[2].split()[1])
    i = lines.index("tauA1")
    tauA1 = np.array([[float(v) for v in lines[i + 1 + r].split()] for r in range(s)])
    j = lines.index("A2")
    A2g = np.array([[float(v) for v in lines[j + 1 + r].split()] for r in range(s)])
    A1, A2, ae = bk.dirk_window([[0.0, 0.0], [1.0 - theta, theta]], s, tau)
    assert A1.shape == (s, s) and np.allclose(A1 * tau, tauA1, rtol=0, atol=1e-15)
    assert np.array_equal(A2, A2g) and np.array_equal(ae, [1.0 - theta])


@pytest.mark.parametrize("tab,s", [("sdirk2", 1), ("sdirk2", 4), ("sdirk3", 2), ("sdirk3", 8)])
def test_sdirk_windows_solve_the_sequential_steps(bk, tab, s):
    """No explicit stage: A2 = I_s (x) A, A1 = I/tau with -1/tau couplings to the previous step's last
    stage; the all-at-once Kronecker solve (oracle O8) with these matrices equals classical
    sequential stepping."""
    A_tab = synth.SDIRK2 if tab == "sdirk2" else synth.SDIRK3
    tau = 0.05
    A1, A2, ae = bk.dirk_window(A_tab, s, tau)
    m = len(A_tab)
    assert A1.shape == (s * m, s * m) and not ae.any()
    K = synth.convdiff2d(6, tau=float("inf"), gamma=1.0)
    N, mass = K.n_rows, (1.0 / 6) ** 2
    rng = np.random.default_rng(5)
    y0 = rng.uniform(-1, 1, N)
    B = rng.uniform(-1, 1, (N, s * m))
    B0 = np.zeros((N, s * m))
    B0[:, :m] = (mass / tau * y0)[:, None]
    Ya = oracle.dirk_all_at_once(K, mass, A1, A2, B, B0)
    Ys = oracle.dirk_sequential(K, mass, A_tab, B, y0, tau, s)
    assert np.abs(Ya - Ys).max() <= 1e-12 * np.abs(Ys).max()


def test_eliminated_stage_window_solves_theta_stepping(bk):
    """Explicit first stage eliminated: with the library's A1, A2 and B0 column 0 =
    M y^n / tau + (1 - Theta)(b^n - K y^n), the all-at-once solve equals s steps of the
    closed-form Theta scheme (oracle.theta_stepping)."""
    tau, theta, s = 0.05, 0.5, 3
    K = synth.convdiff2d(6, tau=float("inf"), gamma=1.0)
    Kd = oracle._dense(K)
    N, mass = K.n_rows, (1.0 / 6) ** 2
    rng = np.random.default_rng(3)
    f, g, y0 = rng.uniform(-1, 1, N), rng.uniform(-1, 1, N), rng.uniform(-1, 1, N)
    b = np.stack([math.sin(1.0 + q * tau) * f + g for q in range(s + 1)], 1)
    A1, A2, ae = bk.dirk_window([[0.0, 0.0], [1.0 - theta, theta]], s, tau)
    B0 = np.zeros((N, s))
    B0[:, 0] = mass / tau * y0 + ae[0] * (b[:, 0] - Kd @ y0)
    Ya = oracle.dirk_all_at_once(K, mass, A1, A2, b[:, 1:], B0)
    Yt = oracle.theta_stepping(K, mass, theta, b, y0, tau, s)
    assert np.abs(Ya - Yt).max() <= 1e-12 * np.abs(Yt).max()


def test_window_rejects_bad_tableaux(bk):
    with pytest.raises(bk.BkError):
        bk.dirk_window([[0.5, 0.1], [0.5, 0.5]], 2, 0.1)            # not lower triangular
    with pytest.raises(bk.BkError):
        bk.dirk_window([[0.0, 0.0], [0.5, 0.0]], 2, 0.1)            # a second explicit stage
    with pytest.raises(bk.BkError):
        bk.dirk_window([[0.0]], 2, 0.1)                             # nothing implicit left
    with pytest.raises(bk.BkError):
        bk.dirk_window(synth.SDIRK2, 2, 0.0)                        # tau <= 0
    with pytest.raises(bk.BkError):
        bk.dirk_window(synth.SDIRK3, 11, 0.1)                       # k = 33 > 32
