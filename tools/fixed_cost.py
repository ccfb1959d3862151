"""Fixed cost of the narrow passes: block_gram / block_update at k = 1, 4 for n = 1 ... c2 size,
one launch between two events vs 20 back-to-back launches (per-launch mean).

    python tools/fixed_cost.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402


def timed(fn, batch, reps=7):
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)          # keep the GPU busy while the host enqueues
        a.record(st)
        for _ in range(batch):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / batch)
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def main():
    ctx = bk.Context(0)
    for k in (1, 4):
        for n in (1, 1000, 100000, 1048576):
            X = synth.multivector(n, k, 3, device="cuda")
            Y = synth.multivector(n, k, 4, device="cuda")
            C = synth.small_dense(k, k, 6, device="cuda")
            G = torch.empty(k, k, dtype=torch.float64, device="cuda")
            row = {"k": k, "n": n}
            for name, fn in (("gram", lambda: bk.block_gram(ctx, X, Y, G)),
                             ("update", lambda: bk.block_update(ctx, Y, X, C, a=1.0, s=1e-3)),
                             ("torch_dot", lambda: torch.sum(X * Y))):
                row[name + "_1"] = round(timed(fn, 1), 2)
                row[name + "_20"] = round(timed(fn, 20), 2)
            print(json.dumps(row))


if __name__ == "__main__":
    main()
