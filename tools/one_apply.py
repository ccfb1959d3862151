"""One configuration of bspmm_apply, launched a few times (for ncu captures).

    python tools/one_apply.py [--cfg c2] [--k 16] [--reps 3] [--coupled]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c2")
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--coupled", action="store_true")
a = ap.parse_args()
ctx = bk.Context(0)
A = synth.make_matrix(a.cfg, device="cuda")
M = bk.Matrix.from_csr(ctx, A)
print(M.info())
X = synth.multivector(A.n_rows, a.k, 3, device="cuda")
Y = torch.empty_like(X)
C = synth.small_dense(a.k, a.k, 6).cuda() if a.coupled else None
for _ in range(a.reps):
    bk.bspmm_apply(ctx, M, X, Y, C=C)
torch.cuda.synchronize()
print("ok")
