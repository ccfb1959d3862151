"""GPU parity at the BENCHMARK sizes (BASELINE.json configs c2-c5), in the launch
configuration bench.py times.  The persistent kernels run many tiles per CTA here,
so their TMA rings wrap (mbarrier phase flips, empty-slot waits, the CG tail's
stage write-back) under an oracle comparison -- the c1 parity cases never do.

  * fused block BiCGStab (k = 8, 12, 16) and fused block CG (k = 8, 16) on c2
    (1 048 576 rows), BiCGStab k = 12 on c3 (2 097 152 rows): the iterate after 10
    fixed iterations vs the oracle O4 / O6, relative Frobenius difference <= 1e-10
    (R18(iv));
  * streaming Gram / update kernels with >= 3 tiles per CTA (ring wraps), R17 bar;
  * apply at c4 k = 16 and c5 k = 8 / 16 / 32 under the default dispatch (c5
    k = 16: y-slab tile order with S = 4): sampled rows against the oracle O1 on the
    sampled rows' CSR sub-problem (rows are independent, so the sample is exact).
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


def _num_sms():
    return torch.cuda.get_device_properties(0).multi_processor_count


def check_close(got, ref, scale, tol=1e-12, what=""):
    err = np.abs(np.asarray(got) - np.asarray(ref))
    bad = err > tol * np.asarray(scale) + 1e-300
    assert not bad.any(), f"{what}: {bad.sum()} entries exceed tol; max err/scale = " \
                          f"{np.max(err / (np.asarray(scale) + 1e-300)):.3e}"


# ----------------------------------------------------------------------------- fused solvers, 10 iterations
_MATS = {}


def _matrix(name):
    """c2 (nonsymmetric), c2s (its symmetric v = 0 variant, for CG), c3; built on the GPU."""
    if name not in _MATS:
        _MATS.clear()
        if name == "c2":
            A = synth.make_matrix("c2", device="cuda")
        elif name == "c2s":
            A = synth.convdiff2d(1024, v=(0.0, 0.0), device="cuda")
        else:
            A = synth.make_matrix(name, device="cuda")
        _MATS[name] = (A, A.to("cpu"))
    return _MATS[name]


@pytest.mark.parametrize("method,cfg,k", [("bicgstab", "c2", 8), ("bicgstab", "c2", 12), ("bicgstab", "c2", 16),
                                          ("cg", "c2s", 8), ("cg", "c2s", 16), ("bicgstab", "c3", 12)])
def test_fused_solver_iterate_at_benchmark_size(ctx, bk, method, cfg, k):
    Ag, Ac = _matrix(cfg)
    n = Ag.n_rows
    B = synth.multivector(n, k, synth.SEEDS["B"], device="cuda")
    M = bk.Matrix.from_csr(ctx, Ag)
    X = torch.zeros(n, k, dtype=torch.float64, device="cuda")
    st, rep = bk.block_krylov_solve(ctx, M, B, X, method=method, rtol=1e-30, max_iters=10, x0_is_zero=True,
                                    check_every=10, timing=True)
    assert rep["iterations"] == 10, rep
    assert rep["n_class"]["fused_tail"] == 10, rep["n_class"]      # the fused passes ran
    if cfg in ("c2", "c2s"):                                           # 2-D: reductions in the applies
        assert rep["n_class"]["fused_apply"] == 10, rep["n_class"]
        assert rep["n_class"]["fused_apply_dots"] == (10 if method == "bicgstab" else 0), rep["n_class"]
    Xr, rr = oracle.SOLVERS[method](Ac, B.cpu(), rtol=1e-30, max_iters=10)
    Xg = X.cpu().numpy()
    rel = np.linalg.norm(Xg - Xr) / np.linalg.norm(Xr)
    assert rel <= 1e-10, (method, cfg, k, rel)
    # per-column too: no column may be off even if the Frobenius norm hides it
    relc = np.linalg.norm(Xg - Xr, axis=0) / np.linalg.norm(Xr, axis=0)
    assert np.all(relc <= 1e-10), relc


def test_fused_tail_ring_wraps_at_c2(ctx, bk):
    """The precondition of the tests above: at c2 the fused tails have several tiles per CTA."""
    n, k = 1024 * 1024, 16
    stage = 48 * 1024
    T = (stage // (5 * k * 8)) & ~7                     # bcg tail: 5 operands per tile row
    tiles = -(-n // T)
    assert tiles >= 3 * 2 * _num_sms(), (T, tiles)


# ----------------------------------------------------------------------------- streaming Gram / update, ring wrap
@pytest.mark.parametrize("ka,kb", [(8, 8), (16, 16), (12, 12), (4, 4), (16, 8), (32, 32), (1, 1)])
def test_stream_gram_ring_wraps(ctx, bk, ka, kb):
    T = max(8, min(1024, ((48 * 1024) // (8 * (ka + kb))) & ~7))
    n = 3 * 2 * _num_sms() * T + 777                     # >= 3 tiles per CTA + a ragged tail
    X = synth.multivector(n, ka, 3, device="cuda")
    Y = synth.multivector(n, kb, 4, device="cuda")
    G = torch.empty(ka, kb, dtype=torch.float64, device="cuda")
    bk.block_gram(ctx, X, Y, G)
    Xc, Yc = X.cpu(), Y.cpu()
    ref = oracle.gram(Xc, Yc)
    scale = oracle.gram(Xc.abs(), Yc.abs())
    check_close(G.cpu().numpy(), ref, scale, what=f"gram n={n} {ka}x{kb}")
    Gs = torch.empty(ka, ka, dtype=torch.float64, device="cuda")          # symmetric X^T X
    bk.block_gram(ctx, X, X, Gs)
    check_close(Gs.cpu().numpy(), oracle.gram(Xc, Xc), oracle.gram(Xc.abs(), Xc.abs()), what="gram XtX")


@pytest.mark.parametrize("kp,k", [(8, 8), (16, 16), (12, 12), (4, 4), (1, 1), (32, 32)])
def test_stream_update_ring_wraps(ctx, bk, kp, k):
    T = max(8, min(1024, ((48 * 1024) // (8 * (kp + k))) & ~7))
    n = 3 * 2 * _num_sms() * T + 333
    X0 = synth.multivector(n, k, 3, device="cuda")
    P = synth.multivector(n, kp, 5, device="cuda")
    C = synth.small_dense(kp, k, 6, device="cuda")
    X0c, Pc, Cc = X0.cpu(), P.cpu(), C.cpu()
    for a, s in ((1.0, 1.0), (0.0, -1.0)):
        X = X0.clone()
        bk.block_update(ctx, X, P, C, a=a, s=s)
        ref = oracle.update(X0c, Pc, Cc, a, s)
        scale = abs(a) * X0c.abs().numpy() + abs(s) * (Pc.abs().numpy() @ Cc.abs().numpy())
        check_close(X.cpu().numpy(), ref, scale, what=f"update n={n} {kp}x{k} a={a}")


# ----------------------------------------------------------------------------- c4 / c5 apply, sampled rows
def _sample_rows(n, shape3, rng, count=6000):
    """Random rows + the first / last rows of every z-plane and y-slab boundary lines."""
    nx, ny, nz = shape3
    plane = nx * ny
    special = [0, 1, n - 1, n - 2]
    for z in (0, 1, nz // 2, nz - 1):
        special += [z * plane, z * plane + nx - 1, (z + 1) * plane - 1, (z + 1) * plane - nx]
        for ys in range(0, ny, max(1, ny // 8)):            # y-slab boundaries (S <= 8)
            special += [z * plane + ys * nx, z * plane + ys * nx - 1 if ys else z * plane]
    rows = np.concatenate([rng.integers(0, n, count), np.array(special, dtype=np.int64)])
    return np.unique(rows[(rows >= 0) & (rows < n)])


def _sampled_reference(A, X, rows, C=None, alpha=1.0, beta=0.0, Y0=None):
    """Oracle O1 on the sub-problem: the sampled rows' CSR entries, columns renumbered onto the
    unique X rows they reference (gathered on the device, then copied to the host).
    Returns (reference, componentwise scale |alpha| |A| |X| |C| + |beta| |Y0|)."""
    dev = A.row_ptr.device
    r = torch.from_numpy(rows).to(dev)
    rp = A.row_ptr.to(torch.int64)
    s, e = rp[r], rp[r + 1]
    cnt = e - s
    base = torch.repeat_interleave(s - torch.cumsum(cnt, 0) + cnt, cnt)
    pos = base + torch.arange(int(cnt.sum()), device=dev)
    cols = A.col[pos].to(torch.int64)
    vals = A.val[pos]
    uniq, inv = torch.unique(cols, return_inverse=True)
    sub_rp = torch.zeros(len(rows) + 1, dtype=torch.int64, device=dev)
    sub_rp[1:] = torch.cumsum(cnt, 0)
    Xs = X[uniq].cpu()
    S = synth.Csr(len(rows), len(uniq), sub_rp.to(torch.int32).cpu(), inv.to(torch.int32).cpu(), vals.cpu())
    Sa = synth.Csr(len(rows), len(uniq), S.row_ptr, S.col, S.val.abs())
    Ys = None if Y0 is None else Y0[r].cpu()
    ref = oracle.spmm(S, Xs, C, alpha, beta, Ys)
    scale = abs(alpha) * oracle.spmm(Sa, Xs.abs(), None if C is None else C.abs())
    if Ys is not None:
        scale = scale + abs(beta) * Ys.abs().numpy()
    return ref, scale


@pytest.mark.parametrize("cfg,k", [("c4", 16), ("c5", 8), ("c5", 16), ("c5", 32)])
def test_full_size_3d_apply_default_dispatch(ctx, bk, cfg, k):
    A = synth.make_matrix(cfg, device="cuda")
    n = A.n_rows
    X = synth.multivector(n, k, synth.SEEDS["X"], device="cuda")
    M = bk.Matrix.from_csr(ctx, A)
    Y = torch.full((n, k), float("nan"), dtype=torch.float64, device="cuda")
    bk.bspmm_apply(ctx, M, X, Y)
    torch.cuda.synchronize()
    assert not torch.isnan(Y).any(), "rows left unwritten"
    rows = _sample_rows(n, A.shape3, np.random.default_rng(7))
    ref, scale = _sampled_reference(A, X, rows)
    check_close(Y[torch.from_numpy(rows).to("cuda")].cpu().numpy(), ref, scale, what=f"{cfg} k={k}")
    # coupled apply at the config's k (DMMA epilogue), beta != 0
    C = synth.small_dense(k, k, synth.SEEDS["C"], device="cuda")
    Y0 = synth.multivector(n, k, synth.SEEDS["Y"], device="cuda")
    Y.copy_(Y0)
    bk.bspmm_apply(ctx, M, X, Y, C=C, alpha=-1.0, beta=0.5)
    refc, scalec = _sampled_reference(A, X, rows, C=C.cpu(), alpha=-1.0, beta=0.5, Y0=Y0)
    check_close(Y[torch.from_numpy(rows).to("cuda")].cpu().numpy(), refc, scalec, what=f"{cfg} k={k} coupled")
    del A, M, X, Y, Y0
    torch.cuda.empty_cache()


# ----------------------------------------------------------------------------- fused vs unfused iteration counts
def _solve_counts(method, k, fused):
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); import json, torch, synth, paper_2504_02117_b200 as bk; "
            f"c = bk.Context(0); A = synth.make_matrix('c1'); M = bk.Matrix.from_csr(c, A); "
            f"B = synth.multivector(A.n_rows, {k}, 2).cuda(); X = torch.zeros_like(B); "
            f"st, r = bk.block_krylov_solve(c, M, B, X, method={method!r}, rtol=1e-10, max_iters=2000, x0_is_zero=True); "
            f"print(json.dumps([st, r['iterations'], X.cpu().flatten().tolist()]))")
    env = dict(os.environ, BK_FUSED="1" if fused else "0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    st, its, x = json.loads(r.stdout.strip().splitlines()[-1])
    return st, its, np.array(x)


@pytest.mark.parametrize("k", [8, 12, 16])
def test_bicgstab_fused_vs_unfused_iteration_count(k):
    """The fused BiCGStab passes against the unfused kernel sequence on the
    same inputs: the same O6 steps in a different summation order -- solutions within 1e-8 and
    both iteration counts inside the oracle's rounding ensemble."""
    s1, i1, x1 = _solve_counts("bicgstab", k, True)
    s0, i0, x0 = _solve_counts("bicgstab", k, False)
    assert s1 == s0 == 0
    # both counts inside the oracle's one-ulp ensemble range (R18: BiCGStab's count on
    # c1 moves by several iterations under rounding-level perturbations of B)
    import test_gpu_parity as tp
    A = synth.make_matrix("c1")
    lo, hi = tp.oracle_bicgstab_count_range(A, synth.multivector(A.n_rows, k, 2))
    assert lo - 1 <= i1 <= hi + 1 and lo - 1 <= i0 <= hi + 1, (i1, i0, lo, hi)
    assert np.linalg.norm(x1 - x0) / np.linalg.norm(x0) <= 1e-8


# ----------------------------------------------------------------------------- narrow (k <= 4) flat kernels
@pytest.mark.parametrize("ka,kb", [(1, 1), (2, 3), (3, 3), (4, 4), (4, 1), (1, 2)])
def test_flat_gram_narrow(ctx, bk, ka, kb):
    """k <= 4 Grams take the flat grid-stride kernel (flat.cu): R17 bar on random data at c2 size,
    bitwise on integers, bitwise reproducible run to run."""
    n = 1024 * 1024 + 17
    X = synth.multivector(n, ka, 3, device="cuda")
    Y = synth.multivector(n, kb, 4, device="cuda")
    G = torch.empty(ka, kb, dtype=torch.float64, device="cuda")
    bk.block_gram(ctx, X, Y, G)
    G2 = torch.empty_like(G)
    bk.block_gram(ctx, X, Y, G2)
    assert torch.equal(G, G2)
    Xc, Yc = X.cpu(), Y.cpu()
    check_close(G.cpu().numpy(), oracle.gram(Xc, Yc), oracle.gram(Xc.abs(), Yc.abs()), what=f"flat gram {ka}x{kb}")
    Xi = synth.multivector(n, ka, 3, integer=True)
    Gi = torch.empty(ka, ka, dtype=torch.float64, device="cuda")
    bk.block_gram(ctx, Xi.cuda(), Xi.cuda(), Gi)
    ref = (Xi.numpy().astype(np.int64).T @ Xi.numpy().astype(np.int64)).astype(np.float64)
    assert np.array_equal(Gi.cpu().numpy(), ref)


@pytest.mark.parametrize("kp,k", [(1, 1), (2, 2), (4, 4), (1, 3), (4, 1), (3, 2)])
def test_flat_update_narrow(ctx, bk, kp, k):
    n = 1024 * 1024 + 5
    X0 = synth.multivector(n, k, 3, integer=True)
    P = synth.multivector(n, kp, 5, integer=True)
    C = synth.small_dense(kp, k, 6, integer=True)
    for a, s in ((1.0, 1.0), (0.0, -1.0), (2.0, 0.5)):
        X = X0.cuda()
        bk.block_update(ctx, X, P.cuda(), C.cuda(), a=a, s=s)
        assert np.array_equal(X.cpu().numpy(), oracle.update(X0, P, C, a, s)), (kp, k, a, s)


def test_gmres64_full_solve_c3_recipe(ctx, bk):
    """c3's solver (BJ configs[2]: block GMRES, k = 12) run to rtol 1e-10 with restart 64 on the c3
    operator recipe at 24^3 (R16; the oracle's long-double Grams make the 128^3 solve too slow for a
    test): solution within 1e-8 of the oracle O5, block iterations within 1 (R18)."""
    A = synth.diffreact3d(24)
    k = 12
    B = synth.multivector(A.n_rows, k, synth.SEEDS["B"])
    M = bk.Matrix.from_csr(ctx, A)
    X = torch.zeros(A.n_rows, k, dtype=torch.float64, device="cuda")
    st, rep = bk.block_krylov_solve(ctx, M, B.cuda(), X, method="gmres", restart=64, rtol=1e-10, max_iters=2000,
                                    x0_is_zero=True)
    Xr, rr = oracle.block_gmres(A, B, rtol=1e-10, max_iters=2000, restart=64)
    assert st == 0 and rr.converged
    assert abs(rep["iterations"] - rr.iterations) <= 1, (rep["iterations"], rr.iterations)
    assert np.linalg.norm(X.cpu().numpy() - Xr) / np.linalg.norm(Xr) <= 1e-8
    assert np.all(rep["true_relres"] <= 1e-9)
