"""Seeded synthetic inputs shared by the oracle tests and the GPU path.

This module holds NONE of the method's arithmetic (no operator apply, no Gram,
no update, no Krylov step).  It only builds the *inputs* of the hot path:

* counter-based random numbers (SplitMix64, reading R19),
* the finite-volume CSR matrices of BASELINE.json configs c1..c5
  (SURVEY.md §8(d) recipe; readings R9, R14-R16, R20, R21),
* the k x k coupling matrices C of the time-stepping window
  (§2.1 eq. (time-stepping-matrices-multiple-parallel-time-steps),
  P:260-288, reading R24).

Everything is written with torch tensor ops so the same code runs on the CPU
(tests, oracle) and on a CUDA device (bench inputs at full size); parity tests
always generate ONCE and hand identical arrays to both sides.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

# ---------------------------------------------------------------------------
# SplitMix64 counter hash (reading R19).  int64 arithmetic wraps, so
# the bit patterns equal the uint64 reference; >> is made logical by masking.
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLD = _s64(0x9E3779B97F4A7C15)
_MIX1 = _s64(0xBF58476D1CE4E5B9)
_MIX2 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """SplitMix64 finaliser of a counter (int64 tensor, wraps like uint64)."""
    z = x + _GOLD
    z = (z ^ _lsr(z, 30)) * _MIX1
    z = (z ^ _lsr(z, 27)) * _MIX2
    return z ^ _lsr(z, 31)


def splitmix64_py(x: int) -> int:
    """Scalar pure-Python reference of the same hash (used by the pins)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _key(seed: int, stream: int) -> int:
    return _s64(seed ^ ((stream * 0x9E3779B97F4A7C15) & _M64))


def uniform01(seed: int, stream: int, index: torch.Tensor) -> torch.Tensor:
    """u = (h >> 11) * 2^-53 in [0, 1), h = splitmix64(key(seed, stream) + index)."""
    h = splitmix64(index + _key(seed, stream))
    return _lsr(h, 11).to(torch.float64) * (2.0 ** -53)


def uniform_pm1(seed: int, stream: int, index: torch.Tensor) -> torch.Tensor:
    """x = 2u - 1 in [-1, 1)."""
    return 2.0 * uniform01(seed, stream, index) - 1.0


def multivector(n_rows: int, k: int, seed: int, *, stream: int = 0,
                row_begin: int = 0, n_global: int | None = None,
                integer: bool = False, ld: int | None = None,
                device="cpu") -> torch.Tensor:
    """Row-major N x k multivector, entry (i, c) keyed by c * N_global + (row_begin + i).

    Column c is therefore independent of k and of the row partition (prefix
    invariance, R19).  integer=True gives values in {-8, ..., 8}
    (exact-arithmetic parity variant).
    """
    n_global = n_rows if n_global is None else n_global
    ld = k if ld is None else ld
    rows = torch.arange(row_begin, row_begin + n_rows, dtype=torch.int64, device=device)
    cols = torch.arange(k, dtype=torch.int64, device=device)
    idx = cols[None, :] * n_global + rows[:, None]
    if integer:
        h = splitmix64(idx + _key(seed, stream))
        v = (_lsr(h, 11) % 17 - 8).to(torch.float64)
    else:
        v = uniform_pm1(seed, stream, idx)
    if ld == k:
        return v.contiguous()
    out = torch.zeros(n_rows, ld, dtype=torch.float64, device=device)
    out[:, :k] = v
    return out


def small_dense(rows: int, cols: int, seed: int, *, stream: int = 0,
                integer: bool = False, device="cpu") -> torch.Tensor:
    """Row-major rows x cols coupling matrix U(-1,1) (or integers in {-8..8})."""
    idx = torch.arange(rows * cols, dtype=torch.int64, device=device)
    if integer:
        h = splitmix64(idx + _key(seed, stream))
        return (_lsr(h, 11) % 17 - 8).to(torch.float64).reshape(rows, cols)
    return uniform_pm1(seed, stream, idx).reshape(rows, cols)


def normal(seed: int, stream: int, index: torch.Tensor) -> torch.Tensor:
    """Standard normal by Box-Muller on two SplitMix64 streams (R20)."""
    u1 = uniform01(seed, 2 * stream, index)
    u2 = uniform01(seed, 2 * stream + 1, index)
    u1 = torch.clamp(u1, min=2.0 ** -60)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


# ---------------------------------------------------------------------------
# CSR container
# ---------------------------------------------------------------------------
@dataclass
class Csr:
    """CSR with int32 row_ptr/col and float64 values (SPEC S:26-31 invariants)."""
    n_rows: int
    n_cols: int
    row_ptr: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor
    name: str = ""
    shape3: tuple | None = None  # (nx, ny, nz) of the grid, z slowest

    @property
    def nnz(self) -> int:
        return int(self.val.numel())

    def to(self, device) -> "Csr":
        return Csr(self.n_rows, self.n_cols, self.row_ptr.to(device), self.col.to(device),
                   self.val.to(device), self.name, self.shape3)

    def rows(self, r0: int, r1: int) -> "Csr":
        """Row slab [r0, r1) with GLOBAL column ids (for the row partition, §8(e))."""
        p0 = int(self.row_ptr[r0]); p1 = int(self.row_ptr[r1])
        rp = (self.row_ptr[r0:r1 + 1] - p0).to(torch.int32)
        return Csr(r1 - r0, self.n_cols, rp.contiguous(), self.col[p0:p1].contiguous(),
                   self.val[p0:p1].contiguous(), self.name, self.shape3)

    def dense(self) -> torch.Tensor:
        """Dense copy (tiny matrices only)."""
        d = torch.zeros(self.n_rows, self.n_cols, dtype=torch.float64)
        rp = self.row_ptr.cpu(); col = self.col.cpu(); val = self.val.cpu()
        for i in range(self.n_rows):
            for p in range(int(rp[i]), int(rp[i + 1])):
                d[i, int(col[p])] += val[p]
        return d


def _assemble(offsets, vals, masks, n, device, name, shape3) -> Csr:
    """Stack per-direction (value, present) columns into CSR; offsets ascending => sorted cols."""
    V = torch.stack(vals, dim=1)
    Mk = torch.stack(masks, dim=1)
    rows = torch.arange(n, dtype=torch.int64, device=device)
    C = rows[:, None] + torch.tensor(offsets, dtype=torch.int64, device=device)[None, :]
    counts = Mk.sum(dim=1)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    col = C[Mk].to(torch.int32)
    val = V[Mk]
    return Csr(n, n, row_ptr.to(torch.int32), col, val, name, shape3)


def _face_dirs(nx, ny, nz, device):
    """Per cell: list of (offset, neighbour-exists mask, axis, sign) in ascending offset order."""
    n = nx * ny * nz
    r = torch.arange(n, dtype=torch.int64, device=device)
    ix = r % nx
    iy = (r // nx) % ny
    iz = r // (nx * ny)
    dirs = []
    if nz > 1:
        dirs.append((-nx * ny, iz > 0, 2, -1))
    if ny > 1:
        dirs.append((-nx, iy > 0, 1, -1))
    dirs.append((-1, ix > 0, 0, -1))
    dirs.append((0, None, None, None))
    dirs.append((1, ix < nx - 1, 0, +1))
    if ny > 1:
        dirs.append((nx, iy < ny - 1, 1, +1))
    if nz > 1:
        dirs.append((nx * ny, iz < nz - 1, 2, +1))
    return n, (ix, iy, iz), dirs


# ---------------------------------------------------------------------------
# c1 / c2: 2-D linear convection-diffusion, CCFV TPFA + upwind
# (§4.1 P:865-913 operator family; R14, R15)
# ---------------------------------------------------------------------------
SDIRK2_GAMMA = 1.0 - math.sqrt(2.0) / 2.0          # DESIGN.md R10
SDIRK3_GAMMA = 0.43586652150845900                  # DESIGN.md R10


def convdiff2d(n: int, *, D: float = 1.0, v=(1.0, 0.5), tau: float = 0.12,
               gamma: float = SDIRK2_GAMMA, integer: bool = False, device="cpu", ny: int | None = None) -> Csr:
    """J = M/tau + gamma*K on an n x ny cell-centred grid (h = 1/n; ny defaults to n: [0,1]^2).

    K: TPFA diffusion (interior T = D, Dirichlet ghost cell T_b = 2D) plus
    first-order upwind convection with face flux q = h (v . n); inflow
    boundary faces carry u_bc = 0, outflow faces add q to the diagonal.
    M = h^2 I.  integer=True: the exact-arithmetic 4 / -1 stencil variant.
    """
    h = 1.0 / n
    ny = n if ny is None else ny
    N, (ix, iy, _), dirs = _face_dirs(n, ny, 1, device)
    offs, vals, masks = [], [], []
    if integer:
        for off, m, _, _ in dirs:
            offs.append(off)
            if m is None:
                vals.append(torch.full((N,), 4.0, dtype=torch.float64, device=device))
                masks.append(torch.ones(N, dtype=torch.bool, device=device))
            else:
                vals.append(torch.full((N,), -1.0, dtype=torch.float64, device=device))
                masks.append(m)
        return _assemble(offs, vals, masks, N, device, f"convdiff2d_int_{n}x{ny}", (n, ny, 1))
    diag = torch.full((N,), h * h / tau, dtype=torch.float64, device=device)
    Kdiag = torch.zeros(N, dtype=torch.float64, device=device)
    T = D
    for off, m, axis, sgn in dirs:
        if m is None:
            continue
        q = h * v[axis] * sgn
        # interior face
        offs.append(off)
        vals.append(torch.full((N,), gamma * (-T + min(q, 0.0)), dtype=torch.float64, device=device))
        masks.append(m)
        Kdiag += torch.where(m, torch.full_like(Kdiag, T + max(q, 0.0)),
                             torch.full_like(Kdiag, 2.0 * T + max(q, 0.0)))
    diag = diag + gamma * Kdiag
    # insert the diagonal at its sorted position (offset 0)
    pos = sorted(range(len(offs) + 1), key=lambda j: (offs + [0])[j])
    offs2 = [(offs + [0])[j] for j in pos]
    vals2 = [(vals + [diag])[j] for j in pos]
    masks2 = [(masks + [torch.ones(N, dtype=torch.bool, device=device)])[j] for j in pos]
    return _assemble(offs2, vals2, masks2, N, device, f"convdiff2d_{n}x{ny}", (n, ny, 1))


# ---------------------------------------------------------------------------
# c3: 3-D nonlinear diffusion-reaction Newton Jacobian (R16;
# PAPER.md §4.2 P:1030-1035 equation family, Neumann boundary)
# ---------------------------------------------------------------------------
def diffreact3d(n: int, *, tau: float = 1e-3, gamma: float = SDIRK3_GAMMA,
                seed_u: int = 1, integer: bool = False, device="cpu") -> Csr:
    h = 1.0 / n
    N, _, dirs = _face_dirs(n, n, n, device)
    if integer:
        offs, vals, masks = [], [], []
        for off, m, _, _ in dirs:
            offs.append(off)
            if m is None:
                vals.append(torch.full((N,), 6.0, dtype=torch.float64, device=device))
                masks.append(torch.ones(N, dtype=torch.bool, device=device))
            else:
                vals.append(torch.full((N,), -1.0, dtype=torch.float64, device=device))
                masks.append(m)
        return _assemble(offs, vals, masks, N, device, f"diffreact3d_int_{n}", (n, n, n))
    u = uniform01(seed_u, 7, torch.arange(N, dtype=torch.int64, device=device))
    diag = h ** 3 / tau + gamma * h ** 3 * (1.0 - 2.0 * u)
    offs, vals, masks = [], [], []
    for off, m, _, _ in dirs:
        if m is None:
            continue
        nb = torch.clamp(torch.arange(N, device=device) + off, 0, N - 1)
        ub = u[nb]
        Df = 1.0 + 0.5 * (u * u + ub * ub)
        jaa = gamma * h * (Df + u * (u - ub))
        jab = gamma * h * (ub * (u - ub) - Df)
        diag = diag + torch.where(m, jaa, torch.zeros_like(jaa))
        offs.append(off); vals.append(jab); masks.append(m)
    offs.append(0); vals.append(diag); masks.append(torch.ones(N, dtype=torch.bool, device=device))
    pos = sorted(range(len(offs)), key=lambda j: offs[j])
    return _assemble([offs[j] for j in pos], [vals[j] for j in pos], [masks[j] for j in pos],
                     N, device, f"diffreact3d_{n}", (n, n, n))


# ---------------------------------------------------------------------------
# c4 / c5: 3-D Richards-type L-scheme Jacobian (R20, R21;
# van Genuchten-Mualem eq. (RelationshipsThetaK), silt loam P:1331-1335)
# ---------------------------------------------------------------------------
SILT_LOAM = dict(theta_s=0.396, theta_r=0.131, alpha=0.423, n=2.06, K_s=4.96e-2)
L_SCHEME = 4.501e-2
TAU_RICHARDS = 1.0 / 96.0


def vg_theta(psi: torch.Tensor, p=SILT_LOAM) -> torch.Tensor:
    """theta(psi), eq. (RelationshipsThetaK) P:1214-1218."""
    n = p["n"]
    th = p["theta_r"] + (p["theta_s"] - p["theta_r"]) * \
        (1.0 / (1.0 + (-p["alpha"] * torch.clamp(psi, max=0.0)) ** n)) ** ((n - 1.0) / n)
    return torch.where(psi > 0, torch.full_like(psi, p["theta_s"]), th)


def vg_K(psi: torch.Tensor, p=SILT_LOAM) -> torch.Tensor:
    """K(psi), eq. (RelationshipsThetaK) P:1219-1222 (theta/theta_S as written)."""
    n = p["n"]
    r = vg_theta(psi, p) / p["theta_s"]
    return p["K_s"] * r ** 0.5 * (1.0 - (1.0 - r ** (n / (n - 1.0))) ** ((n - 1.0) / n)) ** 2


def gaussian_field(nx, ny, nz, *, seed: int = 1, ell: float = 8.0, trunc: int = 17,
                   device="cpu") -> torch.Tensor:
    """Unit-variance Gaussian random field, covariance ~exp(-r^2/(2 ell^2)) (R20).

    White noise blurred separably by a Gaussian kernel of std ell/sqrt(2)
    truncated at +-trunc cells with periodic wrap, normalised analytically by
    sqrt(sum w^2)^3.  Returned shape (nz, ny, nx), x fastest.
    """
    N = nx * ny * nz
    g = normal(seed, 11, torch.arange(N, dtype=torch.int64, device=device)).reshape(1, 1, N)
    s = ell / math.sqrt(2.0)
    t = torch.arange(-trunc, trunc + 1, dtype=torch.float64, device=device)
    w = torch.exp(-0.5 * (t / s) ** 2)
    norm = math.sqrt(float((w * w).sum())) ** 3
    f = g.reshape(nz, ny, nx)

    def blur(x, dim):
        # periodic wrap: y = sum_t w_t x[(i - t) mod n] along `dim`
        y = torch.zeros_like(x)
        for j, tt in enumerate(range(-trunc, trunc + 1)):
            y += float(w[j]) * torch.roll(x, shifts=tt, dims=dim)
        return y

    for d in (2, 1, 0):
        if f.shape[d] > 1:
            f = blur(f, d)
    return (f / norm).contiguous()


def richards3d(nx: int, ny: int, nz: int, *, sigma: float = 2.0, ell: float = 8.0,
               seed: int = 1, integer: bool = False, device="cpu") -> Csr:
    """J = (L/tau) h^3 I + sum_f T_f (e_a - e_b)(e_a - e_b)^T, exactly symmetric (SPD)."""
    h = 1.0 / nx
    N, (_, _, iz), dirs = _face_dirs(nx, ny, nz, device)
    if integer:
        offs, vals, masks = [], [], []
        for off, m, _, _ in dirs:
            offs.append(off)
            if m is None:
                vals.append(torch.full((N,), 6.0, dtype=torch.float64, device=device))
                masks.append(torch.ones(N, dtype=torch.bool, device=device))
            else:
                vals.append(torch.full((N,), -1.0, dtype=torch.float64, device=device))
                masks.append(m)
        return _assemble(offs, vals, masks, N, device, f"richards3d_int", (nx, ny, nz))
    g = gaussian_field(nx, ny, nz, seed=seed, ell=ell, device=device).reshape(-1)
    kappa = torch.exp(sigma * g)
    zc = (iz.to(torch.float64) + 0.5) / nz
    psi = 1.0 - 3.0 * zc
    kr = vg_K(psi) / SILT_LOAM["K_s"]
    Ks = SILT_LOAM["K_s"]
    diag = torch.full((N,), L_SCHEME / TAU_RICHARDS * h ** 3, dtype=torch.float64, device=device)
    offs, vals, masks = [], [], []
    ar = torch.arange(N, device=device)
    for off, m, _, _ in dirs:
        if m is None:
            continue
        nb = torch.clamp(ar + off, 0, N - 1)
        ka, kb = kappa, kappa[nb]
        harm = 2.0 * ka * kb / (ka + kb)
        Tf = Ks * h * harm * (0.5 * (kr + kr[nb]))
        Tf = torch.where(m, Tf, torch.zeros_like(Tf))
        diag = diag + Tf
        offs.append(off); vals.append(-Tf); masks.append(m)
    offs.append(0); vals.append(diag); masks.append(torch.ones(N, dtype=torch.bool, device=device))
    pos = sorted(range(len(offs)), key=lambda j: offs[j])
    return _assemble([offs[j] for j in pos], [vals[j] for j in pos], [masks[j] for j in pos],
                     N, device, f"richards3d_{nx}x{ny}x{nz}", (nx, ny, nz))


def laplace_mms2d(n: int, device="cpu") -> Csr:
    """-Laplace on [0,1]^2, cell-centred TPFA, homogeneous Dirichlet by ghost cell (no h scaling).

    Rows scaled by 1/h^2 so that A u ~ -Delta u (manufactured-solution pin).
    """
    h = 1.0 / n
    N, _, dirs = _face_dirs(n, n, 1, device)
    offs, vals, masks = [], [], []
    diag = torch.zeros(N, dtype=torch.float64, device=device)
    for off, m, _, _ in dirs:
        if m is None:
            continue
        offs.append(off)
        vals.append(torch.full((N,), -1.0 / (h * h), dtype=torch.float64, device=device))
        masks.append(m)
        diag += torch.where(m, torch.full_like(diag, 1.0 / (h * h)), torch.full_like(diag, 2.0 / (h * h)))
    offs.append(0); vals.append(diag); masks.append(torch.ones(N, dtype=torch.bool, device=device))
    pos = sorted(range(len(offs)), key=lambda j: offs[j])
    return _assemble([offs[j] for j in pos], [vals[j] for j in pos], [masks[j] for j in pos],
                     N, device, f"laplace2d_{n}", (n, n, 1))


def random_csr(n_rows: int, n_cols: int, nnz_per_row: int, seed: int, *, empty_rows=(),
               device="cpu") -> Csr:
    """Unstructured CSR with strictly increasing columns per row (edge-case inputs)."""
    gen = torch.Generator().manual_seed(seed)
    rp = [0]; cols = []; vals = []
    for i in range(n_rows):
        if i in empty_rows:
            rp.append(rp[-1]); continue
        m = min(n_cols, max(1, int(torch.randint(1, 2 * nnz_per_row, (1,), generator=gen))))
        c = torch.randperm(n_cols, generator=gen)[:m].sort().values
        cols.append(c)
        vals.append(torch.rand(m, generator=gen, dtype=torch.float64) * 2 - 1)
        rp.append(rp[-1] + m)
    col = torch.cat(cols).to(torch.int32) if cols else torch.zeros(0, dtype=torch.int32)
    val = torch.cat(vals) if vals else torch.zeros(0, dtype=torch.float64)
    return Csr(n_rows, n_cols, torch.tensor(rp, dtype=torch.int32).to(device), col.to(device),
               val.to(device), f"random_{n_rows}x{n_cols}")


# ---------------------------------------------------------------------------
# Time-stepping window -> k x k coupling C (§2.1, P:223-288, P:357-395;
# DESIGN.md R24).  Data only: the builder of C given to bspmm_apply.
# ---------------------------------------------------------------------------
SDIRK2 = [[SDIRK2_GAMMA, 0.0], [1.0 - SDIRK2_GAMMA, SDIRK2_GAMMA]]
# Alexander's 3-stage SDIRK (R10): c = (g, (1+g)/2, 1), b = last row
_g3 = SDIRK3_GAMMA
_a21 = (1.0 - _g3) / 2.0
_b1 = -(6.0 * _g3 * _g3 - 16.0 * _g3 + 1.0) / 4.0
_b2 = (6.0 * _g3 * _g3 - 20.0 * _g3 + 5.0) / 4.0
SDIRK3 = [[_g3, 0.0, 0.0], [_a21, _g3, 0.0], [_b1, _b2, _g3]]


def window_matrices(A_tab, s: int, tau: float, a_elim=None):
    """A1, A2 in R^{sm x sm} of eq. (time-stepping-matrices-multiple-parallel-time-steps).

    0-based: window step q, stage i; A2 = I_s (x) A; A1 = I/tau plus
    A1[q m + i, q m - 1] = -1/tau for q >= 1.  If an explicit first
    stage was eliminated, ``a_elim`` = (a_21, ..., a_m1) is placed in
    A2 at the positions of the -1 entries of A1.
    """
    m = len(A_tab)
    k = s * m
    A1 = torch.eye(k, dtype=torch.float64) / tau
    A2 = torch.zeros(k, k, dtype=torch.float64)
    At = torch.tensor(A_tab, dtype=torch.float64)
    for q in range(s):
        A2[q * m:(q + 1) * m, q * m:(q + 1) * m] = At
        if q >= 1:
            for i in range(m):
                A1[q * m + i, q * m - 1] = -1.0 / tau
                if a_elim is not None:
                    A2[q * m + i, q * m - 1] = a_elim[i]
    return A1, A2


def coupling_c1() -> torch.Tensor:
    """C = (A2 - beta I)^T for SDIRK2 x 2 steps (k = 4), beta = A2[0,0]."""
    _, A2 = window_matrices(SDIRK2, 2, 0.12)
    beta = float(A2[0, 0])
    return (A2 - beta * torch.eye(4, dtype=torch.float64)).T.contiguous()


INT_TABLEAU4 = [[2, 0, 0, 0], [1, 2, 0, 0], [-3, 1, 2, 0], [2, -1, 3, 2]]   # integer stand-in (bitwise tests)


def window_coupling(k: int, stages: int, *, tau: float = 0.12, integer: bool = False,
                    eliminated: bool = False) -> torch.Tensor:
    """C = (A2 - beta I)^T of a window of k / stages steps of an SDIRK
    scheme with ``stages`` stages (2: SDIRK2, 3: Alexander's SDIRK3, 4: an integer
    lower-triangular stand-in).  ``eliminated`` adds the a_{i1} column of an eliminated
    explicit first stage.  The structured (mostly zero) coupling the paper's
    windows give, next to the dense random ``small_dense`` one."""
    assert k % stages == 0
    tab = {2: SDIRK2, 3: SDIRK3, 4: INT_TABLEAU4}[stages]
    if integer:
        tab = [[float(round(4 * v)) for v in row] for row in tab] if stages != 4 else tab
    a_elim = [float(i + 1) for i in range(stages)] if eliminated else None
    if a_elim is not None and not integer:
        a_elim = [v / 8.0 for v in a_elim]
    _, A2 = window_matrices(tab, k // stages, tau, a_elim=a_elim)
    beta = float(A2[0, 0])
    return (A2 - beta * torch.eye(k, dtype=torch.float64)).T.contiguous()


# ---------------------------------------------------------------------------
# Named configurations (BASELINE.json configs)
# ---------------------------------------------------------------------------
SEEDS = dict(matrix=1, B=2, X=3, Y=4, P=5, C=6)

CONFIGS = {
    "c1": dict(kind="convdiff2d", n=32, k=[4]),
    "c1s": dict(kind="convdiff2d", n=32, k=[4], v=(0.0, 0.0)),
    "c2": dict(kind="convdiff2d", n=1024, k=[1, 2, 4, 8, 16, 32]),
    "c2s": dict(kind="convdiff2d", n=1024, k=[8, 16], v=(0.0, 0.0)),   # symmetric c2 (CG)
    "c3": dict(kind="diffreact3d", n=128, k=[12]),
    "c4": dict(kind="richards3d", shape=(256, 256, 256), k=[16]),
    "c5": dict(kind="richards3d", shape=(512, 512, 256), k=[8, 16, 32]),
}


def make_matrix(cfg: str, *, integer: bool = False, device="cpu", scale: int | None = None) -> Csr:
    """Matrix of a named config; `scale` overrides the grid edge (for downsized tests)."""
    c = CONFIGS[cfg]
    if c["kind"] == "convdiff2d":
        n = scale or c["n"]
        return convdiff2d(n, v=c.get("v", (1.0, 0.5)), integer=integer, device=device)
    if c["kind"] == "diffreact3d":
        n = scale or c["n"]
        return diffreact3d(n, integer=integer, device=device)
    if c["kind"] == "richards3d":
        nx, ny, nz = c["shape"] if scale is None else (scale, scale, max(1, scale * c["shape"][2] // c["shape"][0]))
        return richards3d(nx, ny, nz, integer=integer, device=device)
    raise KeyError(cfg)


def expected_nnz(shape3) -> int:
    """nnz = 5N - 2(nx+ny) in 2-D, 7N - 2(nx ny + ny nz + nx nz) in 3-D."""
    nx, ny, nz = shape3
    N = nx * ny * nz
    if nz == 1:
        return 5 * N - 2 * (nx + ny)
    return 7 * N - 2 * (nx * ny + ny * nz + nx * nz)


# ---------------------------------------------------------------------------
# NEXT-3 (Algorithm 1): seeded fields of the nonlinear diffusion-reaction problem
# (initial state y0 and source field g; the operator itself is method arithmetic and
# lives in oracle/alg1.py and the CUDA kernels, R29)
# ---------------------------------------------------------------------------
def dr_fields(nx: int, ny: int, nz: int, seed: int = 1, device="cpu"):
    """(y0, g): U(0,1) per cell (streams 11, 12), lexicographic x-fastest numbering."""
    idx = torch.arange(nx * ny * nz, dtype=torch.int64, device=device)
    return uniform01(seed, 11, idx), uniform01(seed, 12, idx)
