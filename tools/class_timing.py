"""Per-kernel-class device time of a fixed-iteration block solve (library CUDA events,
bk_solve_opts.timing): ms per launch of each class.
    python tools/class_timing.py [--cfg c2] [--k 16] [--method bicgstab] [--iters 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c2")
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--method", default="bicgstab")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--tag", default="")
a = ap.parse_args()
ctx = bk.Context(0)
A = synth.make_matrix(a.cfg, device="cuda")
M = bk.Matrix.from_csr(ctx, A)
B = synth.multivector(A.n_rows, a.k, 2, device="cuda")
X = torch.zeros_like(B)
for rep_i in range(3):
    st, rep = bk.block_krylov_solve(ctx, M, B, X, method=a.method, rtol=0.0, max_iters=a.iters, x0_is_zero=True,
                                    check_every=a.iters, timing=True)
torch.cuda.synchronize()
out = {c: round(1e3 * rep["t_class_ms"][c] / rep["n_class"][c], 2) for c in rep["t_class_ms"] if rep["n_class"][c]}
print(json.dumps({"tag": a.tag or os.environ.get("BK_WIN_TR", ""), "cfg": a.cfg, "k": a.k, "method": a.method,
                  "us_per_launch": out, "n": {c: rep["n_class"][c] for c in out}}))
