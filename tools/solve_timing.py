"""Per-iteration time of a fixed-iteration block solve (slope over iteration counts).

    python tools/solve_timing.py [--cfg c2] [--k 16] [--method bicgstab] [--iters 5,10,20]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c2")
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--method", default="bicgstab")
ap.add_argument("--iters", default="5,10,20")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--check-every", type=int, default=0, help="0: = iteration count (one poll)")
ap.add_argument("--restart", type=int, default=30)
ap.add_argument("--side-stream", action="store_true", help="run on a non-default torch stream")
a = ap.parse_args()
if a.side_stream:
    torch.cuda.set_stream(torch.cuda.Stream())
ctx = bk.Context(0)
A = synth.make_matrix(a.cfg, device="cuda")
M = bk.Matrix.from_csr(ctx, A)
B = synth.multivector(A.n_rows, a.k, 2, device="cuda")
X = torch.zeros_like(B)
out = {}
for it in [int(x) for x in a.iters.split(",")]:
    ts = []
    for r in range(a.reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bk.block_krylov_solve(ctx, M, B, X, method=a.method, rtol=0.0, max_iters=it, x0_is_zero=True,
                              check_every=a.check_every or it, restart=a.restart)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    out[it] = statistics.median(ts)
its = sorted(out)
slope = (out[its[-1]] - out[its[0]]) / (its[-1] - its[0]) if len(its) > 1 else None
print(json.dumps({"cfg": a.cfg, "k": a.k, "method": a.method, "ms": out, "ms_per_iter_slope": slope}))
