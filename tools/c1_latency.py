"""Latency of full small solves (BASELINE.json configs[0], c1 32x32, k = 4): wall time on the
device (CUDA events), kernel launches and per-class kernel time for several poll periods.

    python tools/c1_latency.py
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

ctx = bk.Context(0)
for cfg, meth, kw in (("c1", "gmres", {"restart": 100}), ("c1s", "cg", {}), ("c1", "bicgstab", {})):
    A = synth.make_matrix(cfg)
    M = bk.Matrix.from_csr(ctx, A)
    B = synth.multivector(A.n_rows, 4, 2, device="cuda")
    X = torch.zeros_like(B)
    for ce, gr in ((1, False), (4, False), (16, False), (1, True), (16, True)):
        if gr and meth == "gmres":
            continue
        ts = []
        for r in range(6):
            torch.cuda.synchronize()
            n0 = bk.kernel_launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st, rep = bk.block_krylov_solve(ctx, M, B, X, method=meth, rtol=1e-10, x0_is_zero=True, check_every=ce,
                                            use_graphs=gr, **kw)
            e1.record()
            torch.cuda.synchronize()
            nl = bk.kernel_launch_count() - n0
            if r:
                ts.append(e0.elapsed_time(e1))
        st, rt = bk.block_krylov_solve(ctx, M, B, X, method=meth, rtol=1e-10, x0_is_zero=True, check_every=ce,
                                       timing=True, **kw)
        print(json.dumps({"cfg": cfg, "method": meth, "check_every": ce, "graphs": gr, "ms": round(statistics.median(ts), 3),
                          "iterations": rep["iterations"], "launches": nl,
                          "us_per_iter": round(1e3 * statistics.median(ts) / max(rep["iterations"], 1), 1),
                          "t_class_ms": {c: round(v, 3) for c, v in rt["t_class_ms"].items() if v},
                          "n_class": {c: v for c, v in rt["n_class"].items() if v}}), flush=True)
