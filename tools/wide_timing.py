"""Strided multi-Gram / multi-update timing (GMRES basis layout: N x (m+1)k, ld = (m+1)k)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402

n, k, m = int(sys.argv[1]) if len(sys.argv) > 1 else 2 * 1024 * 1024, 12, 32
ctx = bk.Context(0)
V = synth.multivector(n, (m + 1) * k, 3, device="cuda")
W = synth.multivector(n, k, 4, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[1:])


for j in (0, 3, 7, 15, 31):
    ka = (j + 1) * k
    G = torch.empty(ka, k, dtype=torch.float64, device="cuda")
    H = synth.small_dense(ka, k, 6, device="cuda") * 1e-3
    tg = timed(lambda: bk.block_gram(ctx, V[:, :ka], W, G))
    tu = timed(lambda: bk.block_update(ctx, W, V[:, :ka], H, a=1.0, s=-1.0))
    bg = 8 * n * (ka + k)
    bu = 8 * n * (ka + 2 * k)
    print(json.dumps({"j": j, "ka": ka, "gram_us": round(tg * 1e3, 1), "gram_gbs": round(bg / tg / 1e6, 1),
                      "upd_us": round(tu * 1e3, 1), "upd_gbs": round(bu / tu / 1e6, 1)}))
