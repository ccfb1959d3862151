"""One strided multi-Gram + multi-update (GMRES basis layout) for ncu captures: python tools/one_wide.py [ka]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

ka = int(sys.argv[1]) if len(sys.argv) > 1 else 96
n, k, m = 2 * 1024 * 1024, 12, 32
ctx = bk.Context(0)
V = synth.multivector(n, (m + 1) * k, 3, device="cuda")
W = synth.multivector(n, k, 4, device="cuda")
G = torch.empty(ka, k, dtype=torch.float64, device="cuda")
H = synth.small_dense(ka, k, 6, device="cuda") * 1e-3
for _ in range(2):
    bk.block_gram(ctx, V[:, :ka], W, G)
    bk.block_update(ctx, W, V[:, :ka], H, a=1.0, s=-1.0)
torch.cuda.synchronize()
print("ok")
