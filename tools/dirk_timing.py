"""NEXT-1 measurement: the DIRK window of s steps x m stages solved as one matrix equation
(bk_dirk_solve: splitting fixed point, block Krylov inner solves with k = s m columns) against
classical sequential stepping on the same GPU (one k = 1 solve per stage, right-hand sides built
with the library's apply / update kernels).  c2-size operator (1024^2 convection-diffusion,
CCFV), SDIRK2, tau = 0.12 (R9).

    python tools/dirk_timing.py [--n 1024] [--s 4] [--method bicgstab] [--rtol 1e-8]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--s", default="2,4,8")
ap.add_argument("--method", default="bicgstab")
ap.add_argument("--rtol", type=float, default=1e-8)
ap.add_argument("--tau", type=float, default=0.12)
ap.add_argument("--sym", action="store_true", help="no convection (symmetric K): CG / Chebyshev allowed")
ap.add_argument("--precond", default="none")
ap.add_argument("--inner-rtol", type=float, default=None,
                help="window inner tolerance (the paper's policy for s > 1: 1e-2, outer 1e-8; default --rtol)")
ap.add_argument("--outer-tol", type=float, default=1e-9)
ap.add_argument("--correction", action="store_true", help="bk_dirk_solve_dc (defect-correction form)")
a = ap.parse_args()
v = (0.0, 0.0) if a.sym else (1.0, 0.5)
irtol = a.rtol if a.inner_rtol is None else a.inner_rtol
dev = torch.device("cuda", 0)
ctx = bk.Context(0)
n, tau = a.n, a.tau
A_tab = synth.SDIRK2
m = len(A_tab)
c = np.array(A_tab).sum(1)
K = bk.Matrix.from_csr(ctx, synth.convdiff2d(n, tau=float("inf"), gamma=1.0, v=v, device=dev))
L = bk.Matrix.from_csr(ctx, synth.convdiff2d(n, tau=tau, gamma=A_tab[0][0], v=v, device=dev))
mass = (1.0 / n) ** 2
N = n * n
fg = synth.multivector(N, 3, 11, device=dev)
f, g, y0 = fg[:, 0].contiguous(), fg[:, 1].contiguous(), fg[:, 2].contiguous()


def stage_source(q, i, e):   # b(t) of stage i of step q, with an independent component (R26)
    return math.sin(1.0 + (q + c[i]) * tau) * f + g + e


for s in [int(x) for x in a.s.split(",")]:
    k = s * m
    E = synth.multivector(N, k, 12, device=dev) * 0.5
    B = torch.stack([stage_source(q, i, E[:, q * m + i]) for q in range(s) for i in range(m)], 1).contiguous()
    B0 = torch.zeros(N, k, dtype=torch.float64, device=dev)
    B0[:, :m] = (mass / tau * y0)[:, None]
    A1, A2 = synth.window_matrices(A_tab, s, tau)
    # ---- window (all stages of s steps at once)
    Y = torch.zeros(N, k, dtype=torch.float64, device=dev)
    bk.dirk_solve(ctx, L, K, mass, tau, A1.numpy(), A2.numpy(), B, B0, Y, max_outer=4 * k, outer_tol=a.outer_tol,
                  method=a.method, rtol=irtol, max_iters=2000, precond=a.precond, correction=a.correction)  # warm-up
    Y.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, rep = bk.dirk_solve(ctx, L, K, mass, tau, A1.numpy(), A2.numpy(), B, B0, Y, max_outer=4 * k,
                            outer_tol=a.outer_tol, method=a.method, rtol=irtol, max_iters=2000, precond=a.precond,
                            correction=a.correction)
    torch.cuda.synchronize()
    t_win = (time.perf_counter() - t0) * 1e3
    # ---- sequential stepping: (M/tau + a_ii K) y_i = M y_n / tau + a_ii b_i + sum_{j<i} a_ij (b_j - K y_j)
    Ys = torch.zeros(N, k, dtype=torch.float64, device=dev)
    KY = torch.empty(N, 1, dtype=torch.float64, device=dev)
    rhs = torch.empty(N, 1, dtype=torch.float64, device=dev)
    inner_seq = 0

    def run_seq():
        global inner_seq
        inner_seq = 0
        yn = y0.clone()
        for q in range(s):
            for i in range(m):
                col = q * m + i
                rhs[:, 0] = mass / tau * yn + A_tab[i][i] * B[:, col]
                for j in range(i):
                    bk.bspmm_apply(ctx, K, Ys[:, q * m + j:q * m + j + 1].contiguous(), KY)
                    rhs[:, 0] += A_tab[i][j] * (B[:, q * m + j] - KY[:, 0])
                x = torch.zeros(N, 1, dtype=torch.float64, device=dev)
                _, r = bk.block_krylov_solve(ctx, L, rhs, x, method=a.method, rtol=a.rtol, max_iters=4000,
                                             x0_is_zero=True, precond=a.precond)
                inner_seq += r["iterations"]
                Ys[:, col] = x[:, 0]
            yn = Ys[:, q * m + m - 1].clone()

    run_seq()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_seq()
    torch.cuda.synchronize()
    t_seq = (time.perf_counter() - t0) * 1e3
    diff = float(torch.linalg.norm(Y - Ys) / torch.linalg.norm(Ys))
    print(json.dumps({"n": n, "s": s, "k": k, "method": a.method, "precond": a.precond, "sym": a.sym,
                      "rtol": a.rtol, "inner_rtol": irtol, "correction": a.correction, "outer_tol": a.outer_tol, "window_status": st,
                      "outer": rep["outer_iterations"], "inner_window": rep["inner_iterations_total"],
                      "window_ms": round(t_win, 2), "inner_sequential": inner_seq,
                      "sequential_ms": round(t_seq, 2), "speedup": round(t_seq / t_win, 2),
                      "rel_diff": diff}), flush=True)
