"""Pins of the CPU oracle against things other than itself (CPU only, `-m "not gpu"`).

Each test names what fixes the value: a closed form, a special case that
reduces to a textbook routine, brute force on tiny inputs, exact integer
arithmetic, an invariant, or a value the paper prints (tests/golden/).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def _dense(A):
    return synth.Csr.dense(A).numpy()


# ----------------------------------------------------------------------------- O1 spmm
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_spmm_kronecker_brute_force(k):
    """vec(A X C) = (C^T (x) A) vec(X)  (generalises P:338-356) on N <= 40, dense kron."""
    A = synth.random_csr(37, 40, 5, seed=11, empty_rows=(3, 17))
    X = synth.multivector(40, k, 3).numpy()
    for C in (None, synth.small_dense(k, k + 1, 6).numpy()):
        Cm = np.eye(k) if C is None else C
        Y = oracle.spmm(A, X, C)
        D = _dense(A)
        vecX = X.T.reshape(-1)                      # column-stacked vec
        vecY = np.kron(Cm.T, D) @ vecX
        ref = vecY.reshape(Cm.shape[1], -1).T
        bound = 1e-14 * (np.abs(D) @ np.abs(X) @ np.abs(Cm)) + 1e-300
        assert np.all(np.abs(Y - ref) <= 8 * bound)


def test_spmm_integer_exact_bitwise():
    """Integer stencil (4/-1) x integers in {-8..8}: every partial sum is exact -> bitwise."""
    A = synth.convdiff2d(24, integer=True)
    X = synth.multivector(A.n_rows, 8, 3, integer=True).numpy()
    D = _dense(A).astype(np.int64)
    ref = (D @ X.astype(np.int64)).astype(np.float64)
    Y = oracle.spmm(A, X)
    assert np.array_equal(Y, ref)
    C = synth.small_dense(8, 8, 6, integer=True).numpy()
    Yc = oracle.spmm(A, X, C, alpha=-1.0)
    refc = -((D @ X.astype(np.int64)) @ C.astype(np.int64)).astype(np.float64)
    assert np.array_equal(Yc, refc)


def test_spmm_k1_is_spmv_and_columns_independent():
    """k = 1 is textbook spMV; each column of the block apply equals its own k=1 apply bitwise."""
    A = synth.make_matrix("c1")
    X = synth.multivector(A.n_rows, 8, 3).numpy()
    Y = oracle.spmm(A, X)
    D = _dense(A)
    for c in range(8):
        y1 = oracle.spmm(A, X[:, c:c + 1])[:, 0]
        assert np.array_equal(Y[:, c], y1)
        assert np.allclose(y1, D @ X[:, c], rtol=0, atol=1e-14 * np.abs(D).sum(1).max())


def test_spmm_duplicated_and_prefix_columns():
    A = synth.make_matrix("c1")
    X4 = synth.multivector(A.n_rows, 4, 3).numpy()
    X8 = synth.multivector(A.n_rows, 8, 3).numpy()
    assert np.array_equal(X8[:, :4], X4)               # prefix invariance of the generator
    Y8 = oracle.spmm(A, X8)
    assert np.array_equal(Y8[:, :4], oracle.spmm(A, X4))
    Xd = np.concatenate([X4, X4], axis=1)
    Yd = oracle.spmm(A, Xd)
    assert np.array_equal(Yd[:, :4], Yd[:, 4:])


def test_spmm_identity_and_spec_examples():
    """S:50 Identity(3)(1,2,3) -> (1,2,3); S:51 [2](3) -> (6); S:69 row (1,2) C^T, C=[[0,1],[1,0]] -> (2,1)."""
    I3 = synth.Csr(3, 3, torch.tensor([0, 1, 2, 3], dtype=torch.int32),
                   torch.tensor([0, 1, 2], dtype=torch.int32), torch.ones(3, dtype=torch.float64))
    assert np.array_equal(oracle.spmm(I3, np.array([[1.0], [2.0], [3.0]]))[:, 0], [1.0, 2.0, 3.0])
    A1 = synth.Csr(1, 1, torch.tensor([0, 1], dtype=torch.int32), torch.tensor([0], dtype=torch.int32),
                   torch.tensor([2.0], dtype=torch.float64))
    assert oracle.spmm(A1, np.array([[3.0]]))[0, 0] == 6.0
    Yrow = oracle.spmm(A1, np.array([[0.5, 1.0]]), C=np.array([[0.0, 1.0], [1.0, 0.0]]).T)
    assert np.array_equal(Yrow, [[2.0, 1.0]])
    X = synth.multivector(3, 4, 5).numpy()
    assert np.array_equal(oracle.spmm(I3, X), X)


def test_spmm_alpha_beta_semantics():
    """Y = alpha A X C + beta Y; beta = 0 must not read Y (NaN garbage is overwritten)."""
    A = synth.make_matrix("c1")
    X = synth.multivector(A.n_rows, 4, 3).numpy()
    Y0 = synth.multivector(A.n_rows, 4, 4).numpy()
    nan = np.full_like(Y0, np.nan)
    Y = oracle.spmm(A, X, alpha=2.0, beta=0.0, Y=nan)
    assert np.all(np.isfinite(Y))
    assert np.array_equal(Y, 2.0 * oracle.spmm(A, X))      # 2x is exact scaling
    Yb = oracle.spmm(A, X, alpha=1.0, beta=-0.5, Y=Y0)
    assert np.allclose(Yb, oracle.spmm(A, X) - 0.5 * Y0, rtol=0, atol=1e-15)


def test_spmm_rows_matches_full():
    A = synth.make_matrix("c1")
    X = synth.multivector(A.n_rows, 4, 3).numpy()
    rows = np.array([0, 1, 31, 32, 500, 1023])
    assert np.array_equal(oracle.spmm_rows(A, rows, X), oracle.spmm(A, X)[rows])


# ----------------------------------------------------------------------------- O2 gram
def test_gram_all_ones_closed_form():
    N = 10007
    X = np.ones((N, 3)); Y = np.ones((N, 2))
    assert np.array_equal(oracle.gram(X, Y), np.full((3, 2), float(N)))


def test_gram_integer_exact():
    X = synth.multivector(5000, 6, 3, integer=True).numpy()
    Y = synth.multivector(5000, 5, 4, integer=True).numpy()
    ref = (X.astype(np.int64).T @ Y.astype(np.int64)).astype(np.float64)
    assert np.array_equal(oracle.gram(X, Y), ref)


def test_gram_close_to_exactly_rounded_sum():
    """Long-double accumulation vs the EXACT rational sum (fractions.Fraction):
    |G - exact| <= 2^-53 |exact| (final rounding) + N 2^-63 sum|x y| (64-bit mantissa steps)."""
    from fractions import Fraction
    N = 3000
    X = synth.multivector(N, 3, 3).numpy()
    Y = synth.multivector(N, 2, 4).numpy()
    G = oracle.gram(X, Y)
    for a in range(3):
        for b in range(2):
            ex = sum((Fraction(float(x)) * Fraction(float(y)) for x, y in zip(X[:, a], Y[:, b])), Fraction(0))
            absum = float(np.sum(np.abs(X[:, a] * Y[:, b])))
            err = abs(Fraction(float(G[a, b])) - ex)
            assert err <= Fraction(2.0 ** -53) * abs(ex) + Fraction(N * 2.0 ** -63 * absum)


def test_gram_symmetric_psd_and_norms():
    """X^T X symmetric PSD; diag = squared column norms."""
    X = synth.multivector(3000, 5, 3).numpy()
    G = oracle.gram(X, X)
    assert np.array_equal(G, G.T)
    assert np.min(np.linalg.eigvalsh(G)) > 0
    for c in range(5):
        assert math.isclose(G[c, c], math.fsum(X[:, c] ** 2), rel_tol=1e-15)


# ----------------------------------------------------------------------------- O3 update
def test_update_special_cases_and_integer_exact():
    X = synth.multivector(777, 4, 3).numpy()
    P = synth.multivector(777, 4, 5).numpy()
    assert np.array_equal(oracle.update(X, P, np.eye(4), 1.0, 1.0), X + P)
    assert np.array_equal(oracle.update(X, P, np.zeros((4, 4)), 2.0, 1.0), 2.0 * X)
    Xi = synth.multivector(777, 4, 3, integer=True).numpy()
    Pi = synth.multivector(777, 6, 5, integer=True).numpy()
    Ci = synth.small_dense(6, 4, 6, integer=True).numpy()
    ref = (3 * Xi.astype(np.int64) - Pi.astype(np.int64) @ Ci.astype(np.int64)).astype(np.float64)
    assert np.array_equal(oracle.update(Xi, Pi, Ci, 3.0, -1.0), ref)
    nan = np.full_like(X, np.nan)
    assert np.all(np.isfinite(oracle.update(nan, P, np.eye(4), 0.0, 1.0)))


# ----------------------------------------------------------------------------- small dense
def test_chol_and_lu_against_lapack_and_breakdown():
    rng = np.random.default_rng(0)
    M = rng.standard_normal((6, 6)); G = M @ M.T + 6 * np.eye(6)
    R = oracle.chol_upper(G, 1e-13)
    assert np.allclose(R, np.linalg.cholesky(G).T, atol=1e-13)
    Rhs = rng.standard_normal((6, 3))
    assert np.allclose(oracle.spd_solve(G, Rhs, 1e-13), np.linalg.solve(G, Rhs), atol=1e-12)
    N = rng.standard_normal((6, 6))
    assert np.allclose(oracle.lu_solve(N, Rhs, 1e-13), np.linalg.solve(N, Rhs), atol=1e-10)
    S = np.ones((3, 3))
    with pytest.raises(oracle.Breakdown):
        oracle.chol_upper(S, 1e-13)
    with pytest.raises(oracle.Breakdown):
        oracle.lu_solve(S, np.ones((3, 1)), 1e-13)


# ----------------------------------------------------------------------------- solvers
def _eye_csr(n):
    return synth.Csr(n, n, torch.arange(n + 1, dtype=torch.int32), torch.arange(n, dtype=torch.int32),
                     torch.ones(n, dtype=torch.float64))


@pytest.mark.parametrize("method", ["cg", "gmres", "bicgstab"])
def test_identity_converges_in_one_iteration(method):
    """A = I converges in one iteration."""
    B = synth.multivector(50, 4, 2).numpy()
    X, rep = oracle.SOLVERS[method](_eye_csr(50), B, rtol=1e-12)
    assert rep.converged and rep.iterations == 1
    assert np.allclose(X, B, atol=1e-14)


@pytest.mark.parametrize("method,cfg", [("cg", "c1s"), ("gmres", "c1"), ("bicgstab", "c1")])
def test_small_systems_match_dense_lu(method, cfg):
    """Brute force: converged block solve equals dense LU within kappa * rtol (c1: kappa ~ 170)."""
    A = synth.make_matrix(cfg)
    B = synth.multivector(A.n_rows, 4, 2).numpy()
    kw = {"restart": 100} if method == "gmres" else {}
    X, rep = oracle.SOLVERS[method](A, B, rtol=1e-10, max_iters=1000, **kw)
    assert rep.converged
    Xd = oracle.dense_solve(A, B)
    assert np.linalg.norm(X - Xd) / np.linalg.norm(Xd) < 200 * 1e-10
    assert np.all(rep.true_relres < 1e-9)


def _scalar_cg(D, b, iters):
    """Textbook scalar CG (Hestenes-Stiefel) on a dense matrix -- independent formulation."""
    x = np.zeros_like(b); r = b.copy(); p = r.copy(); rr = r @ r
    hist = []
    for _ in range(iters):
        Ap = D @ p
        a = rr / (p @ Ap)
        x = x + a * p
        r = r - a * Ap
        rn = r @ r
        hist.append(math.sqrt(rn))
        p = r + (rn / rr) * p
        rr = rn
    return x, np.array(hist)


def test_block_cg_k1_equals_scalar_cg():
    """k = 1 block CG iterates equal scalar CG."""
    A = synth.make_matrix("c1s")
    b = synth.multivector(A.n_rows, 1, 2).numpy()
    X, rep = oracle.block_cg(A, b, rtol=1e-30, max_iters=25)
    x, hist = _scalar_cg(_dense(A), b[:, 0], 25)
    assert np.allclose(X[:, 0], x, rtol=0, atol=1e-11 * np.abs(x).max())
    h = np.array(rep.history)[:, 0] * np.linalg.norm(b)
    assert np.allclose(h, hist, rtol=1e-9)


def _scalar_gmres_history(D, b, iters):
    """Textbook GMRES: Arnoldi (modified Gram-Schmidt) + least squares per step."""
    n = len(b); beta = np.linalg.norm(b)
    V = np.zeros((n, iters + 1)); H = np.zeros((iters + 1, iters))
    V[:, 0] = b / beta
    hist = []
    for j in range(iters):
        w = D @ V[:, j]
        for i in range(j + 1):
            H[i, j] = w @ V[:, i]; w = w - H[i, j] * V[:, i]
        H[j + 1, j] = np.linalg.norm(w); V[:, j + 1] = w / H[j + 1, j]
        e = np.zeros(j + 2); e[0] = beta
        y = np.linalg.lstsq(H[:j + 2, :j + 1], e, rcond=None)[0]
        hist.append(np.linalg.norm(e - H[:j + 2, :j + 1] @ y))
    return np.array(hist)


def test_block_gmres_k1_equals_scalar_gmres():
    A = synth.make_matrix("c1")
    b = synth.multivector(A.n_rows, 1, 2).numpy()
    _, rep = oracle.block_gmres(A, b, rtol=1e-30, max_iters=30, restart=40)
    hist = _scalar_gmres_history(_dense(A), b[:, 0], 30)
    h = np.array(rep.history)[:, 0] * np.linalg.norm(b)
    assert np.allclose(h, hist, rtol=1e-7)


def _scalar_bicgstab(D, b, iters):
    """van der Vorst BiCGStab with beta = -rt.t / rt.v (the block form's beta; SURVEY O6 note)."""
    x = np.zeros_like(b); r = b.copy(); rt = r.copy(); p = r.copy()
    for _ in range(iters):
        v = D @ p
        a = (rt @ r) / (rt @ v)
        s = r - a * v
        t = D @ s
        w = (t @ s) / (t @ t)
        x = x + a * p + w * s
        r = s - w * t
        bta = -(rt @ t) / (rt @ v)
        p = r + bta * (p - w * v)
    return x


def test_block_bicgstab_k1_equals_scalar_bicgstab():
    A = synth.make_matrix("c1")
    b = synth.multivector(A.n_rows, 1, 2).numpy()
    X, _ = oracle.block_bicgstab(A, b, rtol=1e-30, max_iters=20)
    x = _scalar_bicgstab(_dense(A), b[:, 0], 20)
    assert np.allclose(X[:, 0], x, rtol=0, atol=1e-9 * np.abs(x).max())


def test_block_gmres_finite_termination():
    """Unrestarted block GMRES is exact after ceil(N/k) block iterations (N = 24, k = 4 -> 6)."""
    A = synth.random_csr(24, 24, 8, seed=5)
    D = _dense(A) + 10 * np.eye(24)
    rp = [0]; cols = []; vals = []
    for i in range(24):
        nz = np.nonzero(D[i])[0]
        cols += list(nz); vals += list(D[i, nz]); rp.append(len(cols))
    A = synth.Csr(24, 24, torch.tensor(rp, dtype=torch.int32), torch.tensor(cols, dtype=torch.int32),
                  torch.tensor(vals, dtype=torch.float64))
    B = synth.multivector(24, 4, 2).numpy()
    X, rep = oracle.block_gmres(A, B, rtol=1e-13, max_iters=6, restart=6)
    assert rep.iterations <= 6
    assert np.linalg.norm(X - np.linalg.solve(D, B)) / np.linalg.norm(X) < 1e-12


def test_manufactured_solution_second_order():
    """-Laplace u = f, u = sin(a pi x) sin(b pi y) per column; cell-centred TPFA is 2nd order."""
    errs = []
    for n in (16, 32, 64):
        A = synth.laplace_mms2d(n)
        h = 1.0 / n
        xc = (np.arange(n) + 0.5) * h
        Xg, Yg = np.meshgrid(xc, xc)          # row = y * n + x
        cols_u, cols_f = [], []
        for a, b in ((1, 1), (1, 2), (2, 1)):
            u = np.sin(a * np.pi * Xg) * np.sin(b * np.pi * Yg)
            cols_u.append(u.reshape(-1)); cols_f.append(((a * a + b * b) * np.pi ** 2 * u).reshape(-1))
        U = np.stack(cols_u, 1); F = np.stack(cols_f, 1)
        X, rep = oracle.block_cg(A, F, rtol=1e-12, max_iters=2000)
        assert rep.converged
        errs.append(np.sqrt(np.mean((X - U) ** 2, axis=0)))
    errs = np.array(errs)
    order = np.log2(errs[:-1] / errs[1:])
    assert np.all(order > 1.9) and np.all(order < 2.1)


def test_permutation_invariance():
    """Permuted RHS columns give permuted solutions."""
    A = synth.make_matrix("c1s")
    B = synth.multivector(A.n_rows, 4, 2).numpy()
    perm = [2, 0, 3, 1]
    X, _ = oracle.block_cg(A, B, rtol=1e-10)
    Xp, _ = oracle.block_cg(A, B[:, perm], rtol=1e-10)
    assert np.allclose(Xp, X[:, perm], rtol=0, atol=1e-9 * np.abs(X).max())


def test_duplicated_rhs_is_breakdown_status():
    """Rank-deficient block (duplicated columns, cf. shift P:592) -> breakdown status, not a crash."""
    A = synth.make_matrix("c1s")
    b = synth.multivector(A.n_rows, 2, 2).numpy()
    B = np.concatenate([b, b[:, :1]], axis=1)
    _, rep = oracle.block_cg(A, B, rtol=1e-10)
    assert rep.status == "breakdown" and rep.breakdown_column == 2


def test_block_size_helps_iterations():
    """fewer iterations when increasing the block size (SPD, soft invariant)."""
    A = synth.make_matrix("c1s")
    B = synth.multivector(A.n_rows, 8, 2).numpy()
    worst = max(oracle.block_cg(A, B[:, c:c + 1], rtol=1e-8)[1].iterations for c in range(8))
    _, rep = oracle.block_cg(A, B, rtol=1e-8)
    assert rep.converged and rep.iterations <= worst


def test_bicgstab_count_is_rounding_sensitive():
    """Evidence for DESIGN.md R18 (BiCGStab iteration counts): on c1 the oracle's OWN block
    BiCGStab count moves by more than one iteration when the right-hand side is perturbed by one
    ulp -- so no implementation with another summation order can be held to +-1; the GPU tests
    compare against the range of this one-ulp ensemble instead.  (CG / GMRES counts are stable
    and keep +-1.)"""
    A = synth.make_matrix("c1")
    for k in (1, 4):
        B = synth.multivector(A.n_rows, k, 2).numpy()
        its = []
        for sd in range(6):
            noise = np.random.default_rng(sd).uniform(-1, 1, B.shape) * 2.2e-16 if sd else 0.0
            _, r = oracle.block_bicgstab(A, B * (1 + noise), rtol=1e-10, max_iters=2000)
            assert r.converged
            its.append(r.iterations)
        assert max(its) - min(its) >= 2, (k, its)
    B = synth.multivector(A.n_rows, 4, 2).numpy()
    As = synth.make_matrix("c1s")
    cg = []
    for sd in range(4):
        noise = np.random.default_rng(sd).uniform(-1, 1, B.shape) * 2.2e-16 if sd else 0.0
        cg.append(oracle.block_cg(As, B * (1 + noise), rtol=1e-10, max_iters=2000)[1].iterations)
    assert max(cg) - min(cg) <= 1, cg


# ----------------------------------------------------------------------------- O11 single-reduction CG
def test_cg1_iterates_equal_block_cg():
    """O11 is O4 rearranged (exact arithmetic): the iterates after j iterations agree with the
    independently pinned O4 to rounding, at every j (c1s, k = 4)."""
    A = synth.make_matrix("c1s")
    B = synth.multivector(A.n_rows, 4, 2).numpy()
    for j in (1, 2, 5, 10, 20):
        X1, _ = oracle.block_cg1(A, B, rtol=1e-30, max_iters=j)
        X4, _ = oracle.block_cg(A, B, rtol=1e-30, max_iters=j)
        assert np.linalg.norm(X1 - X4) / np.linalg.norm(X4) < 1e-10, j


def test_cg1_k1_equals_scalar_cg_and_dense_lu():
    """k = 1: textbook Hestenes-Stiefel CG residual history; converged block solve = dense LU."""
    A = synth.make_matrix("c1s")
    b = synth.multivector(A.n_rows, 1, 2).numpy()
    X, rep = oracle.block_cg1(A, b, rtol=1e-30, max_iters=25)
    x, hist = _scalar_cg(_dense(A), b[:, 0], 25)
    assert np.allclose(X[:, 0], x, rtol=0, atol=1e-10 * np.abs(x).max())
    h = np.array(rep.history)[:, 0] * np.linalg.norm(b)
    assert np.allclose(h, hist, rtol=1e-8)
    B = synth.multivector(A.n_rows, 8, 2).numpy()
    X, rep = oracle.block_cg1(A, B, rtol=1e-10)
    assert rep.converged
    Xd = oracle.dense_solve(A, B)
    assert np.linalg.norm(X - Xd) / np.linalg.norm(Xd) < 200 * 1e-10
    assert np.all(rep.true_relres < 1e-9)
    _, r4 = oracle.block_cg(A, B, rtol=1e-10)
    assert abs(rep.iterations - r4.iterations) <= 1


def test_cg1_identity_breakdown_and_one_reduction_per_iteration(monkeypatch):
    """A = I: one iteration; duplicated RHS -> breakdown status; exactly two Gram calls
    (R^T R, R^T W: one reduction pass) and one apply per iteration, vs O4's two passes."""
    B = synth.multivector(50, 4, 2).numpy()
    X, rep = oracle.block_cg1(_eye_csr(50), B, rtol=1e-12)
    assert rep.converged and rep.iterations == 1 and np.allclose(X, B, atol=1e-14)
    A = synth.make_matrix("c1s")
    Bd = synth.multivector(A.n_rows, 2, 2).numpy()
    _, rep = oracle.block_cg1(A, np.concatenate([Bd, Bd[:, :1]], axis=1), rtol=1e-10)
    assert rep.status == "breakdown"
    calls = {"gram": 0, "spmm": 0}
    g0, s0 = oracle.gram, oracle.spmm

    def cg(*a, **kw):
        calls["gram"] += 1
        return g0(*a, **kw)

    def cs(*a, **kw):
        calls["spmm"] += 1
        return s0(*a, **kw)
    monkeypatch.setattr(oracle, "gram", cg)
    monkeypatch.setattr(oracle, "spmm", cs)
    Bk = synth.multivector(A.n_rows, 4, 2).numpy()
    _, rep = oracle.block_cg1(A, Bk, rtol=1e-30, max_iters=7)
    # setup: R = B - A X, W = A R, R^T R, R^T W; per iteration W = A R, R^T R, R^T W;
    # _finish: true residual (one apply, one Gram for the column norms)
    assert calls["spmm"] == 2 + 7 + 1 and calls["gram"] == 2 + 2 * 7 + 1
