"""NEXT-3 measurement: Algorithm 1 on the c3 lattice (BASELINE.json configs[2]: 128^3,
3-stage DIRK, tau = 1e-3 (R9)) for windows 1 and m: Newton iterations per stage,
inner iterations, device time per step and per Newton iteration.

    python tools/alg1_timing.py [--n 128] [--steps 2] [--windows 1,3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--windows", default="1,3")
ap.add_argument("--tau", type=float, default=1e-3)
ap.add_argument("--method", default="bicgstab")
ap.add_argument("--rtol", type=float, default=1e-8)
a = ap.parse_args()
ctx = bk.Context(0)
n = a.n
y0, g = synth.dr_fields(n, n, n, 1, device="cuda")
N = n ** 3
h = 1.0 / n
eps = 1e-8 * np.sqrt(N) * h ** 3 / a.tau          # ~1e-8 relative to ||M y / tau||
A = synth.SDIRK3
for w in [int(x) for x in a.windows.split(",")]:
    bk.alg1_run(ctx, n, n, n, a.tau, y0, g, A, 1, w, eps, method=a.method, rtol=a.rtol, max_iters=2000)  # warm
    torch.cuda.synchronize()
    st, its, rep = bk.alg1_run(ctx, n, n, n, a.tau, y0, g, A, a.steps, w, eps, method=a.method, rtol=a.rtol,
                               max_iters=2000)
    print(json.dumps({"n": n, "N": N, "window": w, "steps": a.steps, "status": st, "newton_its": its,
                      "newton_total": rep["newton_iterations_total"], "inner_total": rep["inner_iterations_total"],
                      "inner_breakdowns": rep["inner_breakdowns"], "ms_total": round(rep["t_total_ms"], 2),
                      "ms_per_step": round(rep["t_total_ms"] / a.steps, 2),
                      "ms_per_newton": round(rep["t_total_ms"] / max(1, rep["newton_iterations_total"]), 2)}),
          flush=True)
