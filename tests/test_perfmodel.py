"""Pins of the performance model against the paper's printed closed forms (CPU only)."""
from fractions import Fraction

from paper_2504_02117_b200 import perfmodel as pm

GOLD = __file__.rsplit("/", 1)[0] + "/golden/ai_spbop.txt"


def test_paper_ai_closed_forms_golden():
    """P:31 AI(spMV) = 1/8; P:675 AI(spBOP) = k/(4(k+1)) at the Fig. AIBOP samples; ~1.8x at k = 16."""
    rows = [ln.split() for ln in open(GOLD) if ln.strip() and not ln.startswith("#")]
    assert pm.paper_ai_spmv() == Fraction(1, 8)
    for r in rows:
        if r[0] == "factor_k16_about":
            ratio = pm.paper_ai_spbop(16) / pm.paper_ai_spmv()
            assert abs(float(ratio) - float(r[1])) < 0.1        # "a factor of about 1.8" (exact 32/17)
            assert ratio == Fraction(32, 17)
        else:
            assert pm.paper_ai_spbop(int(r[0])) == Fraction(r[1])
    assert pm.paper_ai_spbop(1) == pm.paper_ai_spmv()           # k = 1 reduces to spMV


def test_paper_ecm_counts():
    """omega = 2kz, beta = 2z + 2kz, tau = z(2+2k)."""
    assert pm.paper_ecm_counts(8, 1000) == (16000, 18000, 18000)


def test_algorithmic_bytes():
    n, nnz = 1048576, 5238784
    # c2 k = 8 -> 201.3 MB, k = 16 -> 335.5 MB, k = 1 -> 83.8 MB
    assert round(pm.spmm_bytes(n, nnz, 8) / 1e6, 1) == 201.3
    assert round(pm.spmm_bytes(n, nnz, 16) / 1e6, 1) == 335.5
    assert round(pm.spmm_bytes(n, nnz, 1) / 1e6, 1) == 83.8
    assert pm.gram_bytes(10, 3, 2) == 8 * 10 * 5 and pm.gram_bytes(10, 3, 3, same=True) == 240
    assert pm.update_bytes(10, 4, 4) == 8 * 10 * 12 and pm.update_bytes(10, 4, 4, a_nonzero=False) == 640
    assert pm.spmm_flops(100, 4) == 800 and pm.spmm_flops(100, 4, 10, coupled=True) == 800 + 320


def test_fused_solver_pass_counts():
    """The solver byte models count the N x k passes solve.cpp enqueues:
    fused BiCGStab = 2 applies + 17 passes (+ 2 for the separate column dots when k does not
    divide 32: T and S read once); fused CG = 1 apply + 11 passes; unfused BiCGStab for k = 3."""
    from paper_2504_02117_b200 import perfmodel as pm
    n, nnz = 1000, 5000
    for k, extra in ((4, 0), (8, 0), (12, 2), (16, 0)):
        v = 8 * n * k
        assert pm.bicgstab_iter_bytes(n, nnz, k) == 2 * pm.spmm_bytes(n, nnz, k) + (17 + extra) * v
    for k in (4, 8, 12, 16):
        assert pm.cg_iter_bytes(n, nnz, k) == pm.spmm_bytes(n, nnz, k) + 11 * 8 * n * k
    assert not pm.bicgstab_fused(3) and not pm.bicgstab_fused(32)
    assert pm.cg_iter_bytes(n, nnz, 3) > pm.spmm_bytes(n, nnz, 3) + 11 * 8 * n * 3
    # single-reduction CG (O11): tail 9 passes + apply (+ 2 for the Gram pass unless the
    # reduction rides in the apply's epilogue)
    for k in (4, 8, 12, 16):
        v = 8 * n * k
        assert pm.cg1_iter_bytes(n, nnz, k, fused_apply=True) == pm.spmm_bytes(n, nnz, k) + 9 * v
        assert pm.cg1_iter_bytes(n, nnz, k) == pm.spmm_bytes(n, nnz, k) + 11 * v
    assert pm.cg1_iter_bytes(n, nnz, 3) == 4 * pm.update_bytes(n, 3, 3) + pm.spmm_bytes(n, nnz, 3) + 2 * 8 * n * 3


def test_bicgstab_solve_bytes_counts_only_enqueued_passes():
    """bench.py's solve bytes: with X0 = 0 and a packed B, R0 = P0 = Rt = B
    are read in place (no copies) and the same-operand column dots read B once -- 1 norm pass
    before and a copy + apply + norm pass after the iterations, nothing more; otherwise the three
    setup copies (R, Rt, P) come back."""
    n, nnz, k = 1000, 5000, 16
    v = 8 * n * k
    it = pm.bicgstab_iter_bytes(n, nnz, k)
    assert pm.bicgstab_solve_bytes(n, nnz, k, 5) == (v + 5 * it + 2 * v
                                                     + pm.spmm_bytes(n, nnz, k, beta_nonzero=True) + v)
    assert pm.bicgstab_solve_bytes(n, nnz, k, 5, rt_is_b=False) == pm.bicgstab_solve_bytes(n, nnz, k, 5) + 6 * v


def test_bicgstab_fused_apply_bytes():
    """One rank, 2-D band plan (solve.cpp fapply): the two reduction passes ride in the applies --
    2 applies + 14 N x k passes per iteration (3 fewer than the fused-pass structure)."""
    n, nnz = 1000, 5000
    for k in (8, 12, 16):
        v = 8 * n * k
        assert pm.bicgstab_iter_bytes(n, nnz, k, fused_apply=True) == 2 * pm.spmm_bytes(n, nnz, k) + 14 * v
        assert pm.bicgstab_iter_bytes(n, nnz, k) - pm.bicgstab_iter_bytes(n, nnz, k, fused_apply=True) == \
            (3 if 32 % k == 0 else 5) * v
