"""GPU parity of the single-reduction block CG (BK_CG1, oracle O11,
DESIGN.md §4.4 / R32) through the C ABI:

  * converged solves on c1s (k = 1, 4, 5, 8, 12, 16, 32: the fused tail for k % 4 == 0,
    k <= 16; the one-pass Gram for the other k <= 16; two Grams at k = 32) -- solution within
    1e-8 of O11, iteration count within 1, and the iterate after 10 fixed iterations within
    1e-10 (R18);
  * the fused passes against the unfused kernel sequence (BK_FUSED=0) on the same inputs;
  * c2 size (1 048 576 rows, the TMA rings wrap): 10 fixed iterations vs O11 at 1e-10, with
    the reduction in the W = A R apply's epilogue (RED 4) and the one-pass tail;
  * CUDA-graph replay bitwise equal to eager launches; A = I; breakdown as a status;
  * the p > 1 pass structure on the loopback transport: ONE allreduce per iteration.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bk():
    import paper_2504_02117_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(bk):
    c = bk.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("k", [1, 4, 5, 8, 12, 16, 32])
def test_cg1_solve_matches_oracle(ctx, bk, k):
    A = synth.make_matrix("c1s")
    B = synth.multivector(A.n_rows, k, 2)
    M = bk.Matrix.from_csr(ctx, A)
    X = torch.zeros(A.n_rows, k, dtype=torch.float64, device="cuda")
    st, rep = bk.block_krylov_solve(ctx, M, B.cuda(), X, method="cg1", rtol=1e-10, max_iters=2000,
                                    x0_is_zero=True)
    Xr, rr = oracle.block_cg1(A, B, rtol=1e-10, max_iters=2000)
    assert rr.converged and rep["converged"] and st == 0, rep
    assert abs(rep["iterations"] - rr.iterations) <= 1, (rep["iterations"], rr.iterations)
    assert np.linalg.norm(X.cpu().numpy() - Xr) / np.linalg.norm(Xr) <= 1e-8
    assert np.all(rep["true_relres"] <= 1e-9)
    Xs, _ = oracle.block_cg1(A, B, rtol=1e-30, max_iters=10)
    X10 = torch.zeros_like(X)
    st, rep10 = bk.block_krylov_solve(ctx, M, B.cuda(), X10, method="cg1", rtol=1e-30, max_iters=10,
                                      x0_is_zero=True)
    assert rep10["iterations"] == 10
    assert np.linalg.norm(X10.cpu().numpy() - Xs) / np.linalg.norm(Xs) <= 1e-10


def test_cg1_nonzero_x0_and_iterates_equal_block_cg(ctx, bk):
    """X0 != 0 path (R = B - A X0); the GPU CG1 iterate after 10 iterations also equals O4's."""
    A = synth.make_matrix("c1s")
    k = 8
    B = synth.multivector(A.n_rows, k, 2)
    X0 = synth.multivector(A.n_rows, k, 3)
    M = bk.Matrix.from_csr(ctx, A)
    X = X0.clone().cuda()
    bk.block_krylov_solve(ctx, M, B.cuda(), X, method="cg1", rtol=1e-30, max_iters=10)
    X4, _ = oracle.block_cg(A, B, X0=X0, rtol=1e-30, max_iters=10)
    X11, _ = oracle.block_cg1(A, B, X0=X0, rtol=1e-30, max_iters=10)
    g = X.cpu().numpy()
    assert np.linalg.norm(g - X11) / np.linalg.norm(X11) <= 1e-10
    assert np.linalg.norm(g - X4) / np.linalg.norm(X4) <= 1e-9


def _solve_sub(k, fused):
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); import json, torch, synth, paper_2504_02117_b200 as bk; "
            f"c = bk.Context(0); A = synth.make_matrix('c1s'); M = bk.Matrix.from_csr(c, A); "
            f"B = synth.multivector(A.n_rows, {k}, 2).cuda(); X = torch.zeros_like(B); "
            f"st, r = bk.block_krylov_solve(c, M, B, X, method='cg1', rtol=1e-10, max_iters=2000, x0_is_zero=True, "
            f"timing=True); print(json.dumps([st, r['iterations'], r['n_class']['fused_tail'], "
            f"X.cpu().flatten().tolist()]))")
    env = dict(os.environ, BK_FUSED="1" if fused else "0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    st, its, nt, x = json.loads(r.stdout.strip().splitlines()[-1])
    return st, its, nt, np.array(x)


@pytest.mark.parametrize("k", [4, 12, 16])
def test_cg1_fused_vs_unfused(k):
    s1, i1, t1, x1 = _solve_sub(k, True)
    s0, i0, t0, x0 = _solve_sub(k, False)
    assert s1 == s0 == 0 and t1 == i1 and t0 == 0, (s1, s0, i1, t1, t0)
    assert abs(i1 - i0) <= 1, (i1, i0)
    assert np.linalg.norm(x1 - x0) / np.linalg.norm(x0) <= 1e-8


@pytest.mark.parametrize("k", [8, 16])
def test_cg1_iterate_at_benchmark_size(ctx, bk, k):
    """c2s (the symmetric 1024^2 operator): >= 3 tiles per CTA in every ring."""
    Ag = synth.convdiff2d(1024, v=(0.0, 0.0), device="cuda")
    Ac = Ag.to("cpu")
    n = Ag.n_rows
    B = synth.multivector(n, k, synth.SEEDS["B"], device="cuda")
    M = bk.Matrix.from_csr(ctx, Ag)
    X = torch.zeros(n, k, dtype=torch.float64, device="cuda")
    st, rep = bk.block_krylov_solve(ctx, M, B, X, method="cg1", rtol=1e-30, max_iters=10, x0_is_zero=True,
                                    check_every=10, timing=True)
    assert rep["iterations"] == 10, rep
    assert rep["n_class"]["fused_tail"] == 10, rep["n_class"]
    assert rep["n_class"]["fused_apply"] == 11, rep["n_class"]     # setup + one per iteration
    Xr, _ = oracle.block_cg1(Ac, B.cpu(), rtol=1e-30, max_iters=10)
    Xg = X.cpu().numpy()
    relc = np.linalg.norm(Xg - Xr, axis=0) / np.linalg.norm(Xr, axis=0)
    assert np.all(relc <= 1e-10), relc


def test_cg1_graph_replay_bitwise(ctx, bk):
    A = synth.make_matrix("c1s")
    B = synth.multivector(A.n_rows, 8, 2).cuda()
    M = bk.Matrix.from_csr(ctx, A)
    X1 = torch.zeros_like(B)
    X2 = torch.zeros_like(B)
    s1, r1 = bk.block_krylov_solve(ctx, M, B, X1, method="cg1", rtol=1e-10, x0_is_zero=True, check_every=7)
    s2, r2 = bk.block_krylov_solve(ctx, M, B, X2, method="cg1", rtol=1e-10, x0_is_zero=True, check_every=7,
                                   use_graphs=True)
    assert s1 == s2 == 0 and r1["iterations"] == r2["iterations"]
    assert torch.equal(X1, X2)


def test_cg1_identity_and_breakdown(ctx, bk):
    n = 3000
    A = synth.Csr(n, n, torch.arange(n + 1, dtype=torch.int32), torch.arange(n, dtype=torch.int32),
                  torch.ones(n, dtype=torch.float64))
    B = synth.multivector(n, 8, 2)
    X = torch.zeros(n, 8, dtype=torch.float64, device="cuda")
    st, rep = bk.block_krylov_solve(ctx, bk.Matrix.from_csr(ctx, A), B.cuda(), X, method="cg1", x0_is_zero=True)
    assert st == 0 and rep["iterations"] == 1
    assert torch.allclose(X.cpu(), B, atol=1e-14)
    A = synth.make_matrix("c1s")
    b = synth.multivector(A.n_rows, 2, 2)
    Bd = torch.cat([b, b[:, :1], b[:, 1:]], dim=1)
    X = torch.zeros(A.n_rows, 4, dtype=torch.float64, device="cuda")
    st, rep = bk.block_krylov_solve(ctx, bk.Matrix.from_csr(ctx, A), Bd.cuda(), X, method="cg1", x0_is_zero=True)
    _, rr = oracle.block_cg1(A, Bd, rtol=1e-10)
    assert rr.status == "breakdown" and st == 3 and rep["breakdown_column"] >= 0, rep


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("k", [4, 8])
def test_cg1_partitioned_one_allreduce_per_iteration(bk, P, k):
    import test_gpu_multirank as mr
    A = synth.make_matrix("c1s")
    rb = mr.bounds(A.n_rows, P)
    B = synth.multivector(A.n_rows, k, 2)

    def fn(r, c):
        r0, r1 = rb[r], rb[r + 1]
        S = A.rows(r0, r1)
        M = bk.Matrix(c, S.row_ptr, S.col, S.val, n_global=A.n_rows, row_begin=r0, n_local=r1 - r0)
        X = torch.zeros(r1 - r0, k, dtype=torch.float64, device="cuda")
        st, rep = bk.block_krylov_solve(c, M, B[r0:r1].cuda(), X, method="cg1", rtol=1e-10, max_iters=2000,
                                        x0_is_zero=True)
        M.close()
        return st, rep, X.cpu().numpy()

    res = mr.run_ranks(bk, P, fn)
    its = {o[1]["iterations"] for o in res}
    assert len(its) == 1 and all(o[0] == 0 for o in res)
    it = its.pop()
    X = np.concatenate([o[2] for o in res])
    Xr, rr = oracle.block_cg1(A, B, rtol=1e-10, max_iters=2000)
    assert abs(it - rr.iterations) <= 1
    assert np.linalg.norm(X - Xr) / np.linalg.norm(Xr) <= 1e-8
    # setup reduction (1) + one per iteration + the final true-residual norms (1)
    assert res[0][1]["n_allreduce"] == it + 2, (res[0][1]["n_allreduce"], it)


@pytest.mark.parametrize("method,cfg,k", [("cg1", "c1s", 8), ("cg1", "c1s", 5), ("cg1", "c2s", 16),
                                          ("cg", "c2s", 16), ("bicgstab", "c2", 16)])
def test_library_byte_count_matches_perfmodel(ctx, bk, method, cfg, k):
    """The library's own alg_bytes counter (bk_solve_report) grows per iteration by exactly the
    host byte model bench.py uses (perfmodel.py)."""
    from paper_2504_02117_b200 import perfmodel as pm
    A = synth.make_matrix(cfg, device="cuda")
    M = bk.Matrix.from_csr(ctx, A)
    B = synth.multivector(A.n_rows, k, 2, device="cuda")
    X = torch.zeros_like(B)
    got = []
    for it in (3, 8):
        st, rep = bk.block_krylov_solve(ctx, M, B, X, method=method, rtol=1e-30, max_iters=it, x0_is_zero=True,
                                        check_every=it)
        assert rep["iterations"] == it
        got.append(rep["alg_bytes"])
    fa = cfg in ("c1", "c1s", "c2", "c2s") and k in (8, 12, 16)   # 2-D band plan: reduction in the apply
    model = {"cg1": pm.cg1_iter_bytes, "cg": pm.cg_iter_bytes, "bicgstab": pm.bicgstab_iter_bytes}[method]
    assert (got[1] - got[0]) == 5 * model(A.n_rows, A.nnz, k, fused_apply=fa), (got, model(A.n_rows, A.nnz, k))
