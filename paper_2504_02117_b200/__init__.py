"""B200-native block-Krylov hot path of arxiv 2504.02117 (vectorised DIRK via block Krylov).

Thin ctypes binding of the C ABI in include/bk.h (libbk.so, sm_100a CUDA).
Argument marshalling only: every numeric step runs in the library's kernels.
There is NO CPU fallback: importing this package fails loudly when libbk.so is
missing, and every call fails when no CUDA device is present.

Same names as the C ABI:  bspmm_apply, block_gram, block_update,
block_krylov_solve  (plus Context / Matrix handles).  Multivectors are
row-major float64 2-D tensors (torch, on the ctx's device or on the host) or
numpy arrays (host); the row stride is passed as the leading dimension.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BK_LIB_PATH") or os.path.join(_HERE, "lib", "libbk.so")   # override: A/B builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2504_02117_b200.build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

BK_OK, BK_ERR_ARG, BK_NOT_CONVERGED, BK_BREAKDOWN = 0, 1, 2, 3
BK_ERR_CUDA, BK_ERR_NCCL, BK_ERR_OOM, BK_ERR_UNSUPPORTED = 4, 5, 6, 7
BK_MAX_K, BK_MAX_KA = 32, 4096
BK_GRAM_ALLREDUCE = 1
METHODS = {"cg": 0, "gmres": 1, "bicgstab": 2, "cg1": 3}
PRECONDS = {"none": 0, "jacobi": 1, "chebyshev": 2}
CONV = {"all": 0, "first": 1}

EXPORTED = ["bk_version", "bk_kernel_launch_count", "bk_status_string", "bk_last_error", "bk_ctx_create", "bk_ctx_set_stream",
            "bk_ctx_synchronize", "bk_ctx_destroy", "bk_get_nccl_unique_id", "bk_ctx_set_comm",
            "bk_ctx_comm_info", "bk_csr_create", "bk_csr_destroy", "bk_csr_get_info", "bspmm_apply",
            "block_gram", "block_update", "bk_solve_opts_default", "block_krylov_solve", "bk_plan_halo",
            "bk_plan_bands", "bk_dirk_solve", "bk_precond_apply", "bk_alg1_run", "bk_dirk_solve_dc",
            "bk_local_hub_create", "bk_local_hub_destroy", "bk_ctx_set_comm_local", "bk_dirk_window", "bk_dirk_b0"]


class SolveOpts(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("max_iters", ctypes.c_int), ("restart", ctypes.c_int),
                ("precond", ctypes.c_int), ("conv_mode", ctypes.c_int), ("x0_is_zero", ctypes.c_int),
                ("check_every", ctypes.c_int), ("use_graphs", ctypes.c_int), ("rtol", ctypes.c_double),
                ("breakdown_tol", ctypes.c_double), ("timing", ctypes.c_int), ("cheb_steps", ctypes.c_int),
                ("cheb_lmin", ctypes.c_double), ("cheb_lmax", ctypes.c_double)]


KCLASSES = ["spmm", "gram", "update", "fused_tail", "fused_gram", "copy", "fused_dots", "fused_apply",
            "fused_apply_dots"]


class SolveReport(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("breakdown_column", ctypes.c_int), ("relres", ctypes.c_double * BK_MAX_K),
                ("true_relres", ctypes.c_double * BK_MAX_K), ("t_total_ms", ctypes.c_double),
                ("n_spmm", ctypes.c_int64), ("n_gram", ctypes.c_int64), ("n_update", ctypes.c_int64),
                ("n_small", ctypes.c_int64), ("n_allreduce", ctypes.c_int64),
                ("t_class_ms", ctypes.c_double * len(KCLASSES)), ("n_class", ctypes.c_int64 * len(KCLASSES)), ("alg_bytes", ctypes.c_int64)]


class CsrInfo(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("n_local", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("n_ghost", ctypes.c_int64), ("n_boundary_rows", ctypes.c_int64),
                ("n_send_rows", ctypes.c_int64), ("n_neighbors", ctypes.c_int),
                ("interior_contiguous", ctypes.c_int), ("n_bands", ctypes.c_int),
                ("band_extra_rows", ctypes.c_int), ("jacobi_gershgorin", ctypes.c_double)]


_P, _I, _I64, _D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
_sig = {
    "bk_version": ([], _I),
    "bk_kernel_launch_count": ([], _I64),
    "bk_status_string": ([_I], ctypes.c_char_p),
    "bk_last_error": ([_P], ctypes.c_char_p),
    "bk_ctx_create": ([ctypes.POINTER(_P), _I, _P], _I),
    "bk_ctx_set_stream": ([_P, _P], _I),
    "bk_ctx_synchronize": ([_P], _I),
    "bk_ctx_destroy": ([_P], _I),
    "bk_get_nccl_unique_id": ([_P], _I),
    "bk_ctx_set_comm": ([_P, _P, _I, _I], _I),
    "bk_ctx_comm_info": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "bk_dirk_window": ([_I, _P, _I, _D, ctypes.POINTER(_I), _P, _P, _P], _I),
    "bk_dirk_b0": ([_P, _P, _D, _D, _I, _P, _I, _P, _P, _P, _I64], _I),
    "bk_local_hub_create": ([ctypes.POINTER(_P), _I], _I),
    "bk_local_hub_destroy": ([_P], _I),
    "bk_ctx_set_comm_local": ([_P, _P, _I], _I),
    "bk_csr_create": ([_P, ctypes.POINTER(_P), _I64, _I64, _I64, _P, _P, _P, _I64], _I),
    "bk_csr_destroy": ([_P], _I),
    "bk_csr_get_info": ([_P, ctypes.POINTER(CsrInfo)], _I),
    "bspmm_apply": ([_P, _P, _I, _P, _I64, _P, _I, _D, _D, _P, _I64], _I),
    "block_gram": ([_P, _I64, _I, _I, _P, _I64, _P, _I64, _P, _I], _I),
    "block_update": ([_P, _I64, _I, _I, _D, _P, _I64, _D, _P, _I64, _P], _I),
    "bk_solve_opts_default": ([ctypes.POINTER(SolveOpts)], None),
    "block_krylov_solve": ([_P, _P, _I, _P, _I64, _P, _I64, ctypes.POINTER(SolveOpts),
                            ctypes.POINTER(SolveReport)], _I),
    "bk_plan_halo": ([_I, _I, _P, _I64, _P, _P, _I64, _P, _P, _P, _P, _P], _I),
    "bk_plan_bands": ([_I64, _P, _P, _I, _P], _I),
    "bk_dirk_solve": ([_P, _P, _P, _D, _D, _I, _P, _P, _P, _P, _I64, _P, _I64, _I, _D, _P, _P], _I),
    "bk_dirk_solve_dc": ([_P, _P, _P, _D, _D, _I, _P, _P, _P, _P, _I64, _P, _I64, _I, _D, _P, _P], _I),
    "bk_precond_apply": ([_P, _P, _I, _P, _P, _I64, _P, _I64], _I),
    "bk_alg1_run": ([_P, _P, _I, _P, _I, _I, _D, _I, _P, _P, _I64, _P, _P], _I),
}
for _n, (_a, _r) in _sig.items():
    _f = getattr(_lib, _n)
    _f.argtypes = _a
    _f.restype = _r


class BkError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_lib.bk_status_string(status).decode()} ({status}): {msg}")
        self.status = status


def version() -> int:
    return _lib.bk_version()


def kernel_launch_count() -> int:
    """Kernels launched by libbk.so in this process so far (bk_kernel_launch_count)."""
    return int(_lib.bk_kernel_launch_count())


# ----------------------------------------------------------------- marshalling
def _is_torch(t):
    return hasattr(t, "data_ptr") and hasattr(t, "is_cuda")


_F64 = []


def _torch_f64():
    if not _F64:
        import torch
        _F64.append(torch.float64)
    return _F64[0]


def _mv(t, name):
    """(pointer, rows, cols, ld) of a row-major float64 2-D tensor / array."""
    if t is None:
        return None, 0, 0, 0
    if _is_torch(t):
        # (hot: a few attribute reads per call -- launches of the narrow kernels are host-bound)
        if t.dtype is not _torch_f64():
            raise TypeError(f"{name}: dtype must be float64, got {t.dtype}")
        sh = t.shape
        if len(sh) != 2:
            raise ValueError(f"{name}: must be 2-D (rows x k)")
        rows, cols = sh
        s0, s1 = t.stride()
        if cols > 1 and s1 != 1:
            raise ValueError(f"{name}: rows must be contiguous (stride(1) == 1)")
        ld = s0 if rows > 1 else cols
        return t.data_ptr(), rows, cols, (ld if ld > cols else cols)
    a = t
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.ndim != 2:
        raise TypeError(f"{name}: expected a float64 2-D numpy array or torch tensor")
    if a.shape[1] > 1 and a.strides[1] != 8:
        raise ValueError(f"{name}: rows must be contiguous")
    ld = a.strides[0] // 8 if a.shape[0] > 1 else a.shape[1]
    return a.ctypes.data, a.shape[0], a.shape[1], max(ld, a.shape[1])


def _arr(t, dtype_np, name):
    """Pointer + keep-alive of a 1-D index/value array (torch cpu/cuda or numpy)."""
    if _is_torch(t):
        import torch
        want = {np.int32: torch.int32, np.float64: torch.float64}[dtype_np]
        if t.dtype != want or not t.is_contiguous():
            t = t.to(want).contiguous()
        return t.data_ptr(), t
    a = np.ascontiguousarray(t, dtype=dtype_np)
    return a.ctypes.data, a


class Context:
    """bk_ctx: a device + stream (default: torch's current stream on that device)."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise BkError(BK_ERR_CUDA, "no CUDA device (this library has no CPU fallback)")
        if stream is None:
            stream = torch.cuda.current_stream(device)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self.device = device
        self._h = _P()
        st = _lib.bk_ctx_create(ctypes.byref(self._h), device, _P(handle))
        if st:
            raise BkError(st, "bk_ctx_create failed")

    @property
    def handle(self):
        return self._h

    def check(self, st, what=""):
        if st not in (BK_OK,):
            raise BkError(st, f"{what}: {_lib.bk_last_error(self._h).decode()}")

    def set_stream(self, stream):
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self.check(_lib.bk_ctx_set_stream(self._h, _P(handle)), "bk_ctx_set_stream")

    def synchronize(self):
        self.check(_lib.bk_ctx_synchronize(self._h), "bk_ctx_synchronize")

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        st = _lib.bk_get_nccl_unique_id(buf)
        if st:
            raise BkError(st, "bk_get_nccl_unique_id")
        return buf.raw

    def set_comm(self, uid: bytes, nranks: int, rank: int):
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        self.check(_lib.bk_ctx_set_comm(self._h, buf, nranks, rank), "bk_ctx_set_comm")

    def set_comm_local(self, hub: "LocalHub", rank: int):
        """Attach this ctx as virtual rank `rank` of an in-process loopback hub (test transport,
        include/bk.h bk_ctx_set_comm_local)."""
        self.check(_lib.bk_ctx_set_comm_local(self._h, hub.handle, rank), "bk_ctx_set_comm_local")

    def comm_info(self):
        n, r = _I(), _I()
        _lib.bk_ctx_comm_info(self._h, ctypes.byref(n), ctypes.byref(r))
        return n.value, r.value

    def close(self):
        if self._h:
            _lib.bk_ctx_destroy(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class LocalHub:
    """bk_local_hub_create: in-process loopback transport for `nranks` virtual ranks (one host
    thread + one Context each); test infrastructure for the row-partitioned path on one GPU."""

    def __init__(self, nranks: int):
        self._h = _P()
        st = _lib.bk_local_hub_create(ctypes.byref(self._h), nranks)
        if st:
            raise BkError(st, "bk_local_hub_create")
        self.nranks = nranks

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            _lib.bk_local_hub_destroy(self._h)
            self._h = _P()


class Matrix:
    """bk_csr: a (row slab of a) CSR matrix copied into library-owned device memory."""

    def __init__(self, ctx: Context, row_ptr, col, val, n_global=None, row_begin=0, n_local=None):
        self.ctx = ctx
        n_local = (len(row_ptr) - 1) if n_local is None else n_local
        n_global = n_local if n_global is None else n_global
        prp, krp = _arr(row_ptr, np.int32, "row_ptr")
        pcol, kcol = _arr(col, np.int32, "col")
        pval, kval = _arr(val, np.float64, "val")
        nnz = len(val)
        self._h = _P()
        ctx.check(_lib.bk_csr_create(ctx.handle, ctypes.byref(self._h), n_global, row_begin, n_local,
                                     _P(prp), _P(pcol), _P(pval), nnz), "bk_csr_create")
        self.n_global, self.row_begin, self.n_local, self.nnz = n_global, row_begin, n_local, nnz

    @classmethod
    def from_csr(cls, ctx, A, row_begin=0, n_global=None):
        """From any object with row_ptr/col/val/n_rows (e.g. synth.Csr)."""
        return cls(ctx, A.row_ptr, A.col, A.val, n_global=n_global or A.n_cols, row_begin=row_begin,
                   n_local=A.n_rows)

    def info(self) -> dict:
        i = CsrInfo()
        self.ctx.check(_lib.bk_csr_get_info(self._h, ctypes.byref(i)), "bk_csr_get_info")
        return {f: getattr(i, f) for f, _ in CsrInfo._fields_}

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            _lib.bk_csr_destroy(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------- the four calls
def bspmm_apply(ctx: Context, A: Matrix, X, Y, C=None, alpha: float = 1.0, beta: float = 0.0, k=None,
                k_out=None):
    """Y = alpha (A X) C + beta Y   (include/bk.h a1).  Returns Y."""
    px, nx, kx, ldx = _mv(X, "X")
    py, ny, ky, ldy = _mv(Y, "Y")
    pc, _, kc, _ = _mv(C, "C")
    k = kx if k is None else k
    k_out = (kc if C is not None else k) if k_out is None else k_out
    if nx < A.n_local or ny < A.n_local:
        raise ValueError("X / Y have fewer rows than the local matrix")
    ctx.check(_lib.bspmm_apply(ctx.handle, A.handle, k, _P(px), ldx, _P(pc), k_out, float(alpha), float(beta),
                               _P(py), ldy), "bspmm_apply")
    return Y


def block_gram(ctx: Context, X, Y, G, allreduce: bool = False, n=None, ka=None, kb=None):
    """G = X^T Y  (include/bk.h a3), G ka x kb row-major.  Returns G."""
    px, nx, kx, ldx = _mv(X, "X")
    py, ny, ky, ldy = _mv(Y, "Y")
    pg, _, _, _ = _mv(G, "G")
    n = min(nx, ny) if n is None else n
    ctx.check(_lib.block_gram(ctx.handle, n, ka or kx, kb or ky, _P(px), ldx, _P(py), ldy, _P(pg),
                              BK_GRAM_ALLREDUCE if allreduce else 0), "block_gram")
    return G


def block_update(ctx: Context, X, P, C, a: float = 1.0, s: float = 1.0, n=None, kp=None, k=None):
    """X = a X + s P C  in place (include/bk.h a5).  Returns X."""
    px, nx, kx, ldx = _mv(X, "X")
    pp, npr, kpp, ldp = _mv(P, "P")
    pc, _, _, _ = _mv(C, "C")
    n = min(nx, npr) if n is None else n
    ctx.check(_lib.block_update(ctx.handle, n, kp or kpp, k or kx, float(a), _P(px), ldx, float(s), _P(pp), ldp,
                                _P(pc)), "block_update")
    return X


def solve_opts(method="cg", rtol=1e-10, max_iters=1000, restart=30, precond="none", conv_mode="all",
               x0_is_zero=False, check_every=1, breakdown_tol=1e-13, use_graphs=False, timing=False,
               cheb_steps=4, cheb_lmin=0.0, cheb_lmax=0.0) -> SolveOpts:
    o = SolveOpts()
    _lib.bk_solve_opts_default(ctypes.byref(o))
    o.method = METHODS[method]
    o.rtol = rtol
    o.max_iters = max_iters
    o.restart = restart
    o.precond = PRECONDS[precond]
    o.conv_mode = CONV[conv_mode]
    o.x0_is_zero = int(bool(x0_is_zero))
    o.check_every = check_every
    o.breakdown_tol = breakdown_tol
    o.use_graphs = int(bool(use_graphs))
    o.timing = int(bool(timing))
    o.cheb_steps = int(cheb_steps)
    o.cheb_lmin = float(cheb_lmin or 0.0)
    o.cheb_lmax = float(cheb_lmax or 0.0)
    return o


def block_krylov_solve(ctx: Context, A: Matrix, B, X, **opts):
    """Solve A X = B (include/bk.h a6); X holds X0 on entry.  Returns (status, report dict)."""
    pb, nb, kb, ldb = _mv(B, "B")
    px, nx, kx, ldx = _mv(X, "X")
    if kb != kx:
        raise ValueError("B and X must have the same number of columns")
    o = solve_opts(**opts)
    rep = SolveReport()
    st = _lib.block_krylov_solve(ctx.handle, A.handle, kb, _P(pb), ldb, _P(px), ldx, ctypes.byref(o),
                                 ctypes.byref(rep))
    if st not in (BK_OK, BK_NOT_CONVERGED, BK_BREAKDOWN):
        ctx.check(st, "block_krylov_solve")
    k = kb
    out = {"status": {0: "ok", 2: "not_converged", 3: "breakdown"}[rep.status],
           "iterations": rep.iterations, "converged": bool(rep.converged),
           "breakdown_column": rep.breakdown_column, "relres": np.array(rep.relres[:k]),
           "true_relres": np.array(rep.true_relres[:k]), "t_total_ms": rep.t_total_ms,
           "n_spmm": rep.n_spmm, "n_gram": rep.n_gram, "n_update": rep.n_update, "n_small": rep.n_small,
           "n_allreduce": rep.n_allreduce,
           "t_class_ms": {c: rep.t_class_ms[i] for i, c in enumerate(KCLASSES)},
           "n_class": {c: rep.n_class[i] for i, c in enumerate(KCLASSES)}, "alg_bytes": rep.alg_bytes}
    return st, out


def precond_apply(ctx: Context, A: Matrix, R, Z, precond="chebyshev", cheb_steps=4, cheb_lmin=0.0, cheb_lmax=0.0):
    """Z = M^-1 R (bk_precond_apply, NEXT-4): none / jacobi / chebyshev."""
    pr, nr, kr, ldr = _mv(R, "R")
    pz, nz, kz, ldz = _mv(Z, "Z")
    if kr != kz or nr != nz:
        raise ValueError("R and Z must have the same shape")
    o = solve_opts(precond=precond, cheb_steps=cheb_steps, cheb_lmin=cheb_lmin, cheb_lmax=cheb_lmax)
    ctx.check(_lib.bk_precond_apply(ctx.handle, A.handle, kr, ctypes.byref(o), _P(pr), ldr, _P(pz), ldz),
              "bk_precond_apply")
    return Z


class DrProblem(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64), ("tau", ctypes.c_double),
                ("y0", ctypes.c_void_p), ("g", ctypes.c_void_p)]


class Alg1Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("stages_accepted", ctypes.c_int),
                ("newton_iterations_total", ctypes.c_int), ("inner_iterations_total", ctypes.c_int),
                ("inner_breakdowns", ctypes.c_int), ("failed_stage", ctypes.c_int), ("last_norm", ctypes.c_double),
                ("t_total_ms", ctypes.c_double)]


def alg1_run(ctx: Context, nx, ny, nz, tau, y0, g, A_tab, n_steps, window, eps, *, max_newton=50, traj=None,
             **inner):
    """Algorithm 1 (bk_alg1_run, NEXT-3).  y0, g: N-vectors (torch, host or device).  traj:
    optional N x n_steps output (torch, host or device).  Returns (status, newton its per stage,
    report dict)."""
    import torch
    y0 = y0.contiguous()
    g = g.contiguous()
    for t, nm in ((y0, "y0"), (g, "g")):
        if t.dtype != torch.float64 or t.numel() != nx * ny * nz:
            raise ValueError(f"{nm} must be float64 with nx*ny*nz entries")
    A = np.ascontiguousarray(np.asarray(A_tab, dtype=np.float64))
    m = A.shape[0]
    pb = DrProblem(nx, ny, nz, float(tau), y0.data_ptr(), g.data_ptr())
    pt, ldt = (None, 0)
    if traj is not None:
        pt, nt, kt, ldt = _mv(traj, "traj")
    its = (ctypes.c_int * max(1, n_steps * m))()
    o = solve_opts(**inner)
    rep = Alg1Report()
    st = _lib.bk_alg1_run(ctx.handle, ctypes.byref(pb), m, A.ctypes.data, n_steps, window, float(eps), max_newton,
                          ctypes.byref(o), _P(pt), ldt, its, ctypes.byref(rep))
    if st not in (BK_OK, BK_NOT_CONVERGED):
        ctx.check(st, "bk_alg1_run")
    out = {f: getattr(rep, f) for f, _ in Alg1Report._fields_}
    return st, list(its[:n_steps * m]), out


def plan_halo(nranks: int, rank: int, rank_begin, row_ptr, col_global):
    """Host-only halo plan (bk_plan_halo): returns dict(ghost_ids, ghost_owner, col_local, is_boundary)."""
    rb = np.ascontiguousarray(rank_begin, dtype=np.int64)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    cg = np.ascontiguousarray(col_global, dtype=np.int32)
    nnz = len(cg)
    n_local = len(rp) - 1
    gid = np.zeros(max(nnz, 1), dtype=np.int64)
    gown = np.zeros(max(nnz, 1), dtype=np.int32)
    cl = np.zeros(max(nnz, 1), dtype=np.int32)
    bnd = np.zeros(max(n_local, 1), dtype=np.uint8)
    ng = _I64()
    st = _lib.bk_plan_halo(nranks, rank, _P(rb.ctypes.data), n_local, _P(rp.ctypes.data), _P(cg.ctypes.data), nnz,
                           ctypes.byref(ng), _P(gid.ctypes.data), _P(gown.ctypes.data), _P(cl.ctypes.data),
                           _P(bnd.ctypes.data))
    if st:
        raise BkError(st, "bk_plan_halo")
    g = ng.value
    return {"ghost_ids": gid[:g], "ghost_owner": gown[:g], "col_local": cl[:nnz], "is_boundary": bnd[:n_local]}


BK_BAND_MAX = 7


class BandPlan(ctypes.Structure):
    _fields_ = [("nbands", ctypes.c_int32), ("extra_rows", ctypes.c_int32), ("max_row_nnz", ctypes.c_int32),
                ("dmin", ctypes.c_int32 * BK_BAND_MAX), ("dmax", ctypes.c_int32 * BK_BAND_MAX),
                ("width", ctypes.c_int32 * BK_BAND_MAX), ("lo", ctypes.c_int32 * BK_BAND_MAX),
                ("hi", ctypes.c_int32 * BK_BAND_MAX)]


def plan_bands(row_ptr, col, max_extra: int = 96) -> dict:
    """Host-only band plan of the windowed apply (bk_plan_bands): diagonal bands
    [dmin, dmax] of d = col - row and their even-rounded segment bounds lo/hi."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    c = np.ascontiguousarray(col, dtype=np.int32)
    pl = BandPlan()
    st = _lib.bk_plan_bands(len(rp) - 1, _P(rp.ctypes.data), _P(c.ctypes.data), max_extra, ctypes.byref(pl))
    if st:
        raise BkError(st, "bk_plan_bands")
    g = pl.nbands
    return {"nbands": g, "extra_rows": pl.extra_rows, "max_row_nnz": pl.max_row_nnz,
            "dmin": list(pl.dmin[:g]), "dmax": list(pl.dmax[:g]), "width": list(pl.width[:g]),
            "lo": list(pl.lo[:g]), "hi": list(pl.hi[:g])}


def dirk_window(A_tab, s: int, tau: float):
    """Window matrices of s steps of a DIRK tableau (bk_dirk_window, host only): returns
    (A1, A2, a_elim) as numpy arrays (k x k, k x k, m'), k = s m' (m' = m - 1 when the first
    stage is explicit and eliminated)."""
    A = np.ascontiguousarray(np.asarray(A_tab, dtype=np.float64))
    m = A.shape[0]
    A1 = np.zeros((BK_MAX_K, BK_MAX_K))
    A2 = np.zeros((BK_MAX_K, BK_MAX_K))
    ae = np.zeros(max(m, 1))
    k = _I()
    st = _lib.bk_dirk_window(m, A.ctypes.data, int(s), float(tau), ctypes.byref(k), A1.ctypes.data, A2.ctypes.data,
                             ae.ctypes.data)
    if st:
        raise BkError(st, "bk_dirk_window: not a DIRK tableau with at most an explicit first stage, or k > 32")
    kk = k.value
    mi = kk // int(s)
    return (A1.reshape(-1)[:kk * kk].reshape(kk, kk).copy(), A2.reshape(-1)[:kk * kk].reshape(kk, kk).copy(),
            ae[:mi].copy())


def dirk_b0(ctx: Context, K: Matrix, mass: float, tau: float, A_tab, s: int, yn, bn, B0):
    """B0 of the window (bk_dirk_b0): yn, bn (n-vectors or None) and B0 (n x k) host or device."""
    A = np.ascontiguousarray(np.asarray(A_tab, dtype=np.float64))
    keep = []
    if _is_torch(yn):
        py = yn.data_ptr()
    else:
        ya = np.ascontiguousarray(yn, dtype=np.float64)
        keep.append(ya)
        py = ya.ctypes.data
    if bn is None:
        pb = None
    elif _is_torch(bn):
        pb = bn.data_ptr()
    else:
        arr = np.ascontiguousarray(bn, dtype=np.float64)
        keep.append(arr)
        pb = arr.ctypes.data
    p0, n0, k0, ld0 = _mv(B0, "B0")
    ctx.check(_lib.bk_dirk_b0(ctx.handle, K.handle, float(mass), float(tau), A.shape[0], A.ctypes.data, int(s),
                              _P(py), _P(pb), _P(p0), ld0), "bk_dirk_b0")
    return B0


class DirkReport(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("outer_iterations", ctypes.c_int),
                ("inner_iterations_total", ctypes.c_int), ("last_inner_status", ctypes.c_int),
                ("last_change", ctypes.c_double), ("t_total_ms", ctypes.c_double)]


def dirk_solve(ctx: Context, L: Matrix, K: Matrix, mass: float, tau: float, A1, A2, B, B0, Y, *,
               max_outer=None, outer_tol=0.0, correction=False, **inner):
    """NEXT-1 DIRK window (bk_dirk_solve): M Y A1^T + K Y A2^T = B A2^T + B0 by the splitting
    fixed point; `inner` = block_krylov_solve options.  Y: initial guess in, solution out.
    Returns (status, report dict)."""
    pb, nb, kb, ldb = _mv(B, "B")
    p0, n0, k0, ld0 = _mv(B0, "B0")
    py, ny, ky, ldy = _mv(Y, "Y")
    if not (kb == k0 == ky) or ld0 != ldb:
        raise ValueError("B, B0, Y must have the same width; B and B0 the same leading dimension")
    a1 = np.ascontiguousarray(np.asarray(A1, dtype=np.float64))
    a2 = np.ascontiguousarray(np.asarray(A2, dtype=np.float64))
    if a1.shape != (kb, kb) or a2.shape != (kb, kb):
        raise ValueError("A1, A2 must be k x k")
    o = solve_opts(**inner)
    rep = DirkReport()
    fn = _lib.bk_dirk_solve_dc if correction else _lib.bk_dirk_solve
    st = fn(ctx.handle, L.handle, K.handle, float(mass), float(tau), kb, _P(a1.ctypes.data),
                            _P(a2.ctypes.data), _P(pb), _P(p0), ldb, _P(py), ldy,
                            kb if max_outer is None else int(max_outer), float(outer_tol), ctypes.byref(o),
                            ctypes.byref(rep))
    if st not in (BK_OK, BK_NOT_CONVERGED, BK_BREAKDOWN):
        ctx.check(st, "bk_dirk_solve")
    return st, {"status": {0: "ok", 2: "not_converged", 3: "breakdown"}[rep.status],
                "outer_iterations": rep.outer_iterations, "inner_iterations_total": rep.inner_iterations_total,
                "last_change": rep.last_change, "t_total_ms": rep.t_total_ms}
