"""CPU-only checks of the boundary: the C-ABI library loads, exports every symbol
declared in include/bk.h, and its host-only halo planner is correct (no GPU)."""
import os
import re

import numpy as np
import pytest
import torch

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "bk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", src, flags=re.M))
    names.discard("defined")
    return sorted(names)


def test_library_exports_every_declared_symbol():
    import paper_2504_02117_b200 as bk
    decl = _declared_symbols()
    assert {"bspmm_apply", "block_gram", "block_update", "block_krylov_solve"} <= set(decl)
    for name in decl:
        assert hasattr(bk._lib, name), name
    assert set(decl) == set(bk.EXPORTED)
    assert bk.version() == 100


def test_library_is_sm100a_and_links_nccl():
    import subprocess
    import paper_2504_02117_b200 as bk
    out = subprocess.run(["cuobjdump", "--list-elf", bk.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    dyn = subprocess.run(["ldd", bk.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl" in dyn


def test_context_without_gpu_fails_loudly():
    import paper_2504_02117_b200 as bk
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bk.BkError):
        bk.Context(0)


def _partition(n, p):
    b = [n * r // p for r in range(p + 1)]
    return b


@pytest.mark.parametrize("p", [2, 3, 4])
def test_halo_plan_union_equals_global_apply(p):
    """Per-rank apply on renumbered slabs (local cols + gathered ghosts) equals the
    global oracle apply bitwise on integer inputs (SURVEY.md §4 layer 4)."""
    import paper_2504_02117_b200 as bk
    A = synth.richards3d(8, 8, 8, integer=True)
    X = synth.multivector(A.n_rows, 4, 3, integer=True).numpy()
    Yg = oracle.spmm(A, X)
    rb = _partition(A.n_rows, p)
    for r in range(p):
        slab = A.rows(rb[r], rb[r + 1])
        plan = bk.plan_halo(p, r, rb, slab.row_ptr.numpy(), slab.col.numpy())
        assert np.all(np.diff(plan["ghost_ids"]) > 0)
        for gid, own in zip(plan["ghost_ids"], plan["ghost_owner"]):
            assert rb[own] <= gid < rb[own + 1] and own != r
        Xext = np.concatenate([X[rb[r]:rb[r + 1]], X[plan["ghost_ids"]]], axis=0)
        local = synth.Csr(slab.n_rows, Xext.shape[0], slab.row_ptr, torch.from_numpy(plan["col_local"]), slab.val)
        Yr = oracle.spmm(local, Xext)
        assert np.array_equal(Yr, Yg[rb[r]:rb[r + 1]])
        # boundary rows are exactly those touching a ghost column
        rp = slab.row_ptr.numpy()
        for i in range(slab.n_rows):
            touches = np.any(plan["col_local"][rp[i]:rp[i + 1]] >= slab.n_rows)
            assert bool(plan["is_boundary"][i]) == bool(touches)


def test_halo_plan_z_slab_ghosts_are_two_planes():
    """7-point stencil, z-slab partition: ghosts are exactly the plane below and above."""
    import paper_2504_02117_b200 as bk
    nx = ny = 6; nz = 8; p = 4
    A = synth.richards3d(nx, ny, nz, integer=True)
    plane = nx * ny
    rb = [r * (nz // p) * plane for r in range(p + 1)]
    for r in range(p):
        slab = A.rows(rb[r], rb[r + 1])
        plan = bk.plan_halo(p, r, rb, slab.row_ptr.numpy(), slab.col.numpy())
        expect = []
        if r > 0:
            expect += list(range(rb[r] - plane, rb[r]))
        if r < p - 1:
            expect += list(range(rb[r + 1], rb[r + 1] + plane))
        assert list(plan["ghost_ids"]) == expect
        assert int(plan["is_boundary"].sum()) == plane * ((r > 0) + (r < p - 1))


def test_halo_plan_rejects_bad_input():
    import paper_2504_02117_b200 as bk
    with pytest.raises(bk.BkError):
        bk.plan_halo(2, 0, [0, 3, 2], [0, 1], [0])          # decreasing bounds
    with pytest.raises(bk.BkError):
        bk.plan_halo(2, 0, [0, 1, 2], [0, 1], [5])          # column out of range


# ---------------------------------------------------------------- band plan (bk_plan_bands)
def _check_bands(A, plan, max_extra=96):
    """Every nonzero lies in exactly one band; bands are sorted, disjoint (gap > 4),
    lo/hi even with lo <= dmin and hi >= dmax + 1, and extra = sum(hi - lo)."""
    rp = A.row_ptr.numpy().astype(np.int64)
    col = A.col.numpy().astype(np.int64)
    rows = np.repeat(np.arange(A.n_rows), np.diff(rp))
    d = col - rows
    g = plan["nbands"]
    assert 1 <= g <= 7
    dmin, dmax = np.array(plan["dmin"]), np.array(plan["dmax"])
    lo, hi = np.array(plan["lo"]), np.array(plan["hi"])
    assert np.all(dmin <= dmax) and np.all(dmin[1:] > dmax[:-1] + 4)
    assert np.all(lo % 2 == 0) and np.all(hi % 2 == 0) and np.all(lo <= dmin) and np.all(hi >= dmax + 1)
    assert np.all(lo > dmin - 2) and np.all(hi < dmax + 3)
    assert plan["extra_rows"] == int((hi - lo).sum()) <= max_extra
    assert plan["width"] == list(dmax - dmin + 1) and plan["max_row_nnz"] == int((dmax - dmin + 1).sum())
    inband = (d[:, None] >= dmin[None, :]) & (d[:, None] <= dmax[None, :])
    assert np.all(inband.sum(axis=1) == 1)
    assert np.diff(rp).max() <= plan["max_row_nnz"]
    # every distinct offset is covered and each band's ends are attained offsets
    assert set(dmin) | set(dmax) <= set(np.unique(d))


def test_band_plan_2d_3d_stencils():
    """5-point: bands {-nx}, {-1,0,1}, {+nx}; 7-point: also {-nx ny}, {+nx ny}."""
    import paper_2504_02117_b200 as bk
    A = synth.convdiff2d(128)
    p = bk.plan_bands(A.row_ptr, A.col)
    _check_bands(A, p)
    assert p["dmin"] == [-128, -1, 128] and p["dmax"] == [-128, 1, 128]
    assert p["lo"] == [-128, -2, 128] and p["hi"] == [-126, 2, 130] and p["extra_rows"] == 8
    B = synth.diffreact3d(20)
    p = bk.plan_bands(B.row_ptr, B.col)
    _check_bands(B, p)
    assert p["dmin"] == [-400, -20, -1, 20, 400] and p["max_row_nnz"] == 7
    C = synth.richards3d(24, 24, 12)
    _check_bands(C, bk.plan_bands(C.row_ptr, C.col))
    # odd offsets: the +-nx bands of an odd-width grid round outward to even bounds
    O = synth.convdiff2d(25)
    p = bk.plan_bands(O.row_ptr, O.col)
    _check_bands(O, p)
    assert p["lo"] == [-26, -2, 24] and p["hi"] == [-24, 2, 26]


def test_band_plan_rejects_unstructured_and_bad_args():
    import paper_2504_02117_b200 as bk
    R = synth.random_csr(300, 5000, 6, 7, empty_rows=(3, 4))
    assert bk.plan_bands(R.row_ptr, R.col)["nbands"] == 0            # thousands of offsets
    A = synth.convdiff2d(64)
    assert bk.plan_bands(A.row_ptr, A.col, max_extra=4)["nbands"] == 0   # window too wide
    # 9 isolated diagonals -> more than BK_BAND_MAX bands
    n = 200
    offs = [-160, -120, -80, -40, 0, 40, 80, 120, 160]
    rp = [0]; cols = []
    for i in range(n):
        c = [i + o for o in offs if 0 <= i + o < n]
        cols += c; rp.append(len(cols))
    assert bk.plan_bands(rp, cols)["nbands"] == 0
    assert bk.plan_bands([0], [])["nbands"] == 0                       # empty
    with pytest.raises(bk.BkError):
        bk.plan_bands([0, 2, 1], [0, 1])                               # decreasing row_ptr
    with pytest.raises(bk.BkError):
        bk.plan_bands(A.row_ptr, A.col, max_extra=-1)
