"""Pins of the seeded input generators and of the paper's printed values (CPU only)."""
import math

import numpy as np
import pytest
import torch

import synth

GOLD = __file__.rsplit("/", 1)[0] + "/golden/"


def _kv(name):
    out = {}
    for ln in open(GOLD + name):
        ln = ln.split("#")[0].strip()
        if ln:
            k, *v = ln.split()
            out[k] = v
    return out


def test_splitmix64_matches_scalar_reference():
    idx = torch.tensor([0, 1, 2, 12345, 2 ** 40 + 7], dtype=torch.int64)
    h = synth.splitmix64(idx)
    for i, v in zip(idx.tolist(), h.tolist()):
        assert (v & ((1 << 64) - 1)) == synth.splitmix64_py(i)
    # published first output of SplitMix64 seeded with 0 (state advanced once by the golden gamma)
    assert synth.splitmix64_py(0) == 0xE220A8397B1DCDAF


def test_uniform_range_and_moments():
    x = synth.uniform_pm1(2, 0, torch.arange(200000, dtype=torch.int64))
    assert float(x.min()) >= -1.0 and float(x.max()) < 1.0
    assert abs(float(x.mean())) < 5e-3 and abs(float(x.var()) - 1 / 3) < 5e-3


@pytest.mark.parametrize("cfg", ["c1", "c1s", "c3"])
def test_nnz_formula_and_csr_invariants(cfg):
    A = synth.make_matrix(cfg, scale=16 if cfg == "c3" else None)
    assert A.nnz == synth.expected_nnz(A.shape3)
    rp = A.row_ptr.numpy().astype(np.int64); col = A.col.numpy()
    assert rp[0] == 0 and rp[-1] == A.nnz and np.all(np.diff(rp) >= 1)
    for i in range(A.n_rows):
        c = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < A.n_cols


def test_full_size_nnz_c2_c3():
    """Row and nnz counts of BASELINE configs c2, c3."""
    A = synth.make_matrix("c2")
    assert (A.n_rows, A.nnz) == (1048576, 5238784)
    A = synth.make_matrix("c3")
    assert (A.n_rows, A.nnz) == (2097152, 14581760)


def test_c1_is_m_matrix_and_c1s_symmetric():
    D = synth.make_matrix("c1").dense().numpy()
    off = D - np.diag(np.diag(D))
    assert np.all(off <= 0) and np.all(np.diag(D) > 0)
    assert np.all(np.diag(D) >= -off.sum(1))            # weak diagonal dominance by rows
    Ds = synth.make_matrix("c1s").dense().numpy()
    assert np.array_equal(Ds, Ds.T)
    assert np.min(np.linalg.eigvalsh(Ds)) > 0


def test_richards_exactly_symmetric_spd():
    A = synth.richards3d(8, 8, 4)
    D = A.dense().numpy()
    assert np.array_equal(D, D.T)
    assert np.min(np.linalg.eigvalsh(D)) > 0
    assert A.nnz == synth.expected_nnz((8, 8, 4))


def test_van_genuchten_endpoints_and_lipschitz_constant():
    """theta(0) = theta_S, K(0) = K_S; L = max theta'(psi) = 4.501e-2."""
    g = _kv("silt_loam.txt")
    p = dict(theta_s=float(g["theta_s"][0]), theta_r=float(g["theta_r"][0]), alpha=float(g["alpha"][0]),
             n=float(g["n"][0]), K_s=float(g["K_s"][0]))
    assert p == synth.SILT_LOAM
    z = torch.zeros(1, dtype=torch.float64)
    assert float(synth.vg_theta(z)) == p["theta_s"]
    assert math.isclose(float(synth.vg_K(z)), p["K_s"], rel_tol=1e-15)
    psi = torch.linspace(-10, 0, 200001, dtype=torch.float64)
    th = synth.vg_theta(psi)
    L = float(((th[1:] - th[:-1]) / (psi[1:] - psi[:-1])).max())
    assert round(L, 5) == float(g["L"][0])              # 4 significant digits as printed
    assert synth.L_SCHEME == float(g["L"][0])
    assert math.isclose(synth.TAU_RICHARDS, float(g["tau"][0]), rel_tol=1e-15)


def test_theta_method_window_matrices_golden():
    """PAPER.md Example ex:time-stepping-matrices, Theta = 0.5, s = 4."""
    lines = [ln.strip() for ln in open(GOLD + "theta_window.txt") if ln.strip() and not ln.startswith("#")]
    theta = float(lines[0].split()[1]); s = int(lines[1].split()[1]); tau = float(lines[2].split()[1])
    i = lines.index("tauA1")
    tauA1 = np.array([[float(v) for v in lines[i + 1 + r].split()] for r in range(s)])
    j = lines.index("A2")
    A2g = np.array([[float(v) for v in lines[j + 1 + r].split()] for r in range(s)])
    A1, A2 = synth.window_matrices([[theta]], s, tau, a_elim=[1.0 - theta])
    assert np.allclose(A1.numpy() * tau, tauA1, rtol=0, atol=1e-15)
    assert np.array_equal(A2.numpy(), A2g)


def test_sdirk_tableaux_order_conditions():
    """SDIRK2 / SDIRK3 (R10): sum b = 1, b.c = 1/2 (+ b.c^2 = 1/3, b^T A c = 1/6 for order 3)."""
    g = synth.SDIRK2_GAMMA
    A = np.array(synth.SDIRK2); b = A[-1]; c = A.sum(1)
    assert math.isclose(b.sum(), 1.0) and math.isclose(b @ c, 0.5)
    g3 = synth.SDIRK3_GAMMA
    assert abs(g3 ** 3 - 3 * g3 ** 2 + 1.5 * g3 - 1 / 6) < 1e-15
    a21 = (1 - g3) / 2
    b1 = -(6 * g3 ** 2 - 16 * g3 + 1) / 4; b2 = (6 * g3 ** 2 - 20 * g3 + 5) / 4
    A3 = np.array([[g3, 0, 0], [a21, g3, 0], [b1, b2, g3]]); b3 = A3[-1]; c3 = A3.sum(1)
    assert math.isclose(b3.sum(), 1.0, abs_tol=1e-14) and math.isclose(b3 @ c3, 0.5, abs_tol=1e-14)
    assert math.isclose(b3 @ c3 ** 2, 1 / 3, abs_tol=1e-14) and math.isclose(b3 @ A3 @ c3, 1 / 6, abs_tol=1e-14)
    assert np.array_equal(np.array(synth.SDIRK3), A3)                    # the tableau the NEXT-1 driver uses
    assert g == 1 - math.sqrt(2) / 2


def test_coupling_c1_is_split_offdiagonal():
    """C = (A2 - beta I)^T, beta = A2[0,0] (eq. matrix-splitting) for SDIRK2 x 2 steps."""
    C = synth.coupling_c1().numpy()
    g = synth.SDIRK2_GAMMA
    ref = np.zeros((4, 4)); ref[0, 1] = 1 - g; ref[2, 3] = 1 - g
    assert np.array_equal(C, ref)


def test_gaussian_field_unit_variance():
    f = synth.gaussian_field(64, 64, 64, seed=1)
    # correlated field: ~ (64/8)^3 effective samples, so the sample mean fluctuates ~0.1
    assert abs(float(f.mean())) < 0.3 and abs(float(f.std()) - 1.0) < 0.1
