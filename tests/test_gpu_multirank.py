"""The row-partitioned (p > 1) path on ONE GPU, through the library's loopback transport
(include/bk.h bk_local_hub_create / bk_ctx_set_comm_local): P virtual ranks, one host thread
and one Context each.  Everything the NCCL path runs except the NCCL calls themselves
executes here -- bk_csr_create's collective halo plan (ranges allgather, request exchange,
renumbering, interior / boundary split), the halo exchange inside bspmm_apply with the
interior rows on a reduced grid and the ghost-row (GHOST) boundary kernel, the Gram
allreduce, and the solvers' p > 1 pass structure (reductions summed over ranks, the k x k
steps replicated on every rank) -- against the CPU oracle on the global problem
(DESIGN.md §7).
"""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bk():
    import paper_2504_02117_b200 as m
    return m


def run_ranks(bk, P, fn, timeout=600):
    """fn(rank, ctx) on P threads, each with its own stream + Context attached to one hub."""
    hub = bk.LocalHub(P)
    out, err = [None] * P, []

    def body(r):
        try:
            s = torch.cuda.Stream(device=0)
            with torch.cuda.stream(s):
                ctx = bk.Context(0, stream=s)
                ctx.set_comm_local(hub, r)
                out[r] = fn(r, ctx)
                s.synchronize()
                ctx.close()
        except BaseException as e:          # noqa: BLE001 -- reported below
            err.append((r, repr(e)))

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "a rank hung (mismatched collectives)"
    assert not err, err
    hub.close()
    return out


def bounds(n, P, align=1):
    return [((n // align) * r // P) * align for r in range(P)] + [n]


CASES = [(2, "zslab"), (3, "zslab"), (3, "ragged")]


def _partition(A, P, kind):
    nx, ny, nz = A.shape3
    if kind == "zslab":
        return bounds(A.n_rows, P, nx * ny)
    return [0] + [A.n_rows * (2 * r + 1) // (2 * P) + 7 * r for r in range(1, P)] + [A.n_rows]   # mid-plane cuts


@pytest.mark.parametrize("P,kind", CASES)
@pytest.mark.parametrize("k", [1, 4, 12, 16, 32])
def test_partitioned_apply_bitwise(bk, P, kind, k):
    """Union over ranks of the slab applies = the global oracle apply, bitwise (integer data);
    coupled apply with beta too; ghost counts = the halo planes."""
    A = synth.richards3d(12, 10, 9, integer=True)
    rb = _partition(A, P, kind)
    X = synth.multivector(A.n_rows, k, 3, integer=True)
    C = synth.small_dense(k, k, 6, integer=True)
    Y0 = synth.multivector(A.n_rows, k, 4, integer=True)

    def fn(r, ctx):
        r0, r1 = rb[r], rb[r + 1]
        S = A.rows(r0, r1)
        M = bk.Matrix(ctx, S.row_ptr, S.col, S.val, n_global=A.n_rows, row_begin=r0, n_local=r1 - r0)
        Xl = X[r0:r1].cuda()
        Y = torch.full((r1 - r0, k), float("nan"), dtype=torch.float64, device="cuda")
        bk.bspmm_apply(ctx, M, Xl, Y)
        Y2 = Y0[r0:r1].cuda()
        bk.bspmm_apply(ctx, M, Xl, Y2, C=C.cuda(), alpha=-2.0, beta=3.0)
        info = M.info()
        M.close()
        return Y.cpu().numpy(), Y2.cpu().numpy(), info

    res = run_ranks(bk, P, fn)
    assert np.array_equal(np.concatenate([o[0] for o in res]), oracle.spmm(A, X))
    assert np.array_equal(np.concatenate([o[1] for o in res]), oracle.spmm(A, X, C, alpha=-2.0, beta=3.0, Y=Y0))
    plane = 12 * 10
    for r, (_, _, info) in enumerate(res):
        assert info["n_neighbors"] == (r > 0) + (r < P - 1)
        if kind == "zslab":
            assert info["n_ghost"] == info["n_neighbors"] * plane and info["interior_contiguous"] == 1


@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_apply_random_and_gram_allreduce(bk, P):
    """Random data (componentwise 1e-12 bar, R17); block_gram with the allreduce flag gives
    every rank the SAME bits, equal to the global Gram within the bar."""
    A = synth.richards3d(16, 12, 10)
    rb = _partition(A, P, "zslab")
    k = 8
    X = synth.multivector(A.n_rows, k, 3)
    Yr = oracle.spmm(A, X)

    def fn(r, ctx):
        r0, r1 = rb[r], rb[r + 1]
        S = A.rows(r0, r1)
        M = bk.Matrix(ctx, S.row_ptr, S.col, S.val, n_global=A.n_rows, row_begin=r0, n_local=r1 - r0)
        Xl = X[r0:r1].cuda()
        Y = torch.empty(r1 - r0, k, dtype=torch.float64, device="cuda")
        bk.bspmm_apply(ctx, M, Xl, Y)
        G = torch.empty(k, k, dtype=torch.float64, device="cuda")
        bk.block_gram(ctx, Xl, Y, G, allreduce=True)
        M.close()
        return Y.cpu().numpy(), G.cpu().numpy()

    res = run_ranks(bk, P, fn)
    Y = np.concatenate([o[0] for o in res])
    scale = oracle.spmm(synth.Csr(A.n_rows, A.n_cols, A.row_ptr, A.col, A.val.abs()), np.abs(X.numpy()))
    assert np.all(np.abs(Y - Yr) <= 1e-12 * scale + 1e-300)
    Gs = [o[1] for o in res]
    assert all(np.array_equal(Gs[0], g) for g in Gs[1:])                  # identical bits on every rank
    Gr = oracle.gram(X, Yr)
    assert np.all(np.abs(Gs[0] - Gr) <= 1e-12 * oracle.gram(np.abs(X.numpy()), np.abs(Yr)) + 1e-300)


SOLVES = [("cg", "c1s", 4, {}), ("cg", "c1s", 8, {}), ("bicgstab", "c1", 8, {}), ("bicgstab", "c1", 3, {}),
          ("gmres", "c1", 4, {"restart": 100}), ("cg", "c1s", 4, {"precond": "chebyshev", "cheb_steps": 4})]


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("method,cfg,k,kw", SOLVES)
def test_partitioned_solvers_match_oracle(bk, P, method, cfg, k, kw):
    """The solvers' p > 1 path (reductions summed over ranks, replicated k x k steps, halo
    exchanges in every apply and Chebyshev step): the same iteration count on every rank, the
    solution within 1e-8 of the oracle's (R18), CG / GMRES counts within 1 of the oracle's,
    BiCGStab inside its one-ulp ensemble; fused BiCGStab sums each reduction pass with ONE
    allreduce (<= 3 per iteration)."""
    A = synth.make_matrix(cfg)
    rb = bounds(A.n_rows, P)
    B = synth.multivector(A.n_rows, k, 2)

    def fn(r, ctx):
        r0, r1 = rb[r], rb[r + 1]
        S = A.rows(r0, r1)
        M = bk.Matrix(ctx, S.row_ptr, S.col, S.val, n_global=A.n_rows, row_begin=r0, n_local=r1 - r0)
        X = torch.zeros(r1 - r0, k, dtype=torch.float64, device="cuda")
        st, rep = bk.block_krylov_solve(ctx, M, B[r0:r1].cuda(), X, method=method, rtol=1e-10, max_iters=2000,
                                        x0_is_zero=True, **kw)
        M.close()
        return st, rep, X.cpu().numpy()

    res = run_ranks(bk, P, fn)
    its = {o[1]["iterations"] for o in res}
    assert len(its) == 1 and all(o[0] == 0 for o in res), [(o[0], o[1]["iterations"]) for o in res]
    it = its.pop()
    X = np.concatenate([o[2] for o in res])
    Xr, rr = oracle.SOLVERS[method](A, B, rtol=1e-10, max_iters=2000, **kw)
    assert np.linalg.norm(X - Xr) / np.linalg.norm(Xr) <= 1e-8
    if method == "bicgstab":
        import test_gpu_parity as tp
        lo, hi = tp.oracle_bicgstab_count_range(A, B)
        assert lo - 1 <= it <= hi + 1, (it, lo, hi)
        if k % 4 == 0:
            # setup: ||R0|| (1); per iteration [M1 RR] (1) + [RtT ts tt] (1) + ||R||^2 (1); finish: 1
            assert res[0][1]["n_allreduce"] <= 3 * it + 2, res[0][1]["n_allreduce"]
    else:
        assert abs(it - rr.iterations) <= 1, (it, rr.iterations)
    assert np.all(res[0][1]["true_relres"] <= 1e-9)


def test_partitioned_apply_empty_halo_and_host_buffers(bk):
    """A block-diagonal matrix (no ghosts at all) and host X / Y through the partitioned path."""
    n, P, k = 400, 2, 4
    A = synth.Csr(n, n, torch.arange(n + 1, dtype=torch.int32), torch.arange(n, dtype=torch.int32),
                  torch.arange(1, n + 1, dtype=torch.float64))
    X = synth.multivector(n, k, 3)
    rb = bounds(n, P)

    def fn(r, ctx):
        r0, r1 = rb[r], rb[r + 1]
        S = A.rows(r0, r1)
        M = bk.Matrix(ctx, S.row_ptr, S.col, S.val, n_global=n, row_begin=r0, n_local=r1 - r0)
        Yh = np.zeros((r1 - r0, k))
        bk.bspmm_apply(ctx, M, X[r0:r1].numpy(), Yh)
        info = M.info()
        M.close()
        return Yh, info

    res = run_ranks(bk, P, fn)
    assert np.array_equal(np.concatenate([o[0] for o in res]), oracle.spmm(A, X))
    assert all(o[1]["n_ghost"] == 0 for o in res)


@pytest.mark.parametrize("k", [12, 16])
def test_partitioned_apply_slab_order_interior(bk, k):
    """512 x 512 planes split into z-slabs: each rank's interior planes take the y-slab tile order
    (abi.cpp slab_order, also on the p > 1 interior range) -- the union stays bitwise equal to the
    oracle on integer data."""
    A = synth.richards3d(512, 512, 6, integer=True)
    P = 2
    rb = bounds(A.n_rows, P, 512 * 512)
    X = synth.multivector(A.n_rows, k, 3, integer=True)

    def fn(r, ctx):
        r0, r1 = rb[r], rb[r + 1]
        S = A.rows(r0, r1)
        M = bk.Matrix(ctx, S.row_ptr, S.col, S.val, n_global=A.n_rows, row_begin=r0, n_local=r1 - r0)
        Y = torch.full((r1 - r0, k), float("nan"), dtype=torch.float64, device="cuda")
        bk.bspmm_apply(ctx, M, X[r0:r1].cuda(), Y)
        M.close()
        return Y.cpu().numpy()

    res = run_ranks(bk, P, fn)
    assert np.array_equal(np.concatenate(res), oracle.spmm(A, X))
