"""Isolated kernel sweep (L2 flushed before every launch): bspmm / gram / update GB/s vs k.

    python tools/sweep.py [--cfg c2] [--ks 1,2,4,8,16,32] [--ops spmm,gram,update] [--reps 7]
Prints one JSON line per (op, k).  Used for A/B runs of kernel variants
(env BK_SPMM_KERNEL=tile|pipe, BK_SPMM_VEC=2|4|8).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
from paper_2504_02117_b200 import perfmodel as pm  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c2")
    ap.add_argument("--ks", default="1,2,4,8,16,32")
    ap.add_argument("--ops", default="spmm")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--batch", type=int, default=1, help="launches per timed region (amortises host overhead)")
    args = ap.parse_args()
    peak = 6548.8
    dev = torch.device("cuda", 0)
    ctx = bk.Context(0)
    A = synth.make_matrix(args.cfg, device=dev)
    M = bk.Matrix.from_csr(ctx, A)
    n, nnz = A.n_rows, A.nnz
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    flush2 = torch.ones(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    mode = os.environ.get("FLUSH", "wr")

    def do_flush():
        flush.fill_(1.0)                 # write a buffer > L2 ...
        if mode == "wr":
            flush2.sum()                 # ... then read one, so L2 holds clean lines (no write-back in the timed kernel)

    # calibration: plain device copy of 1 GiB (read + write bytes), as MEASURED_PEAKS.json does
    a1 = torch.empty(1 << 27, dtype=torch.float64, device=dev)
    b1 = torch.empty_like(a1)
    ts = []
    for _ in range(5):
        do_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        b1.copy_(a1)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"tag": "copy", "cfg": "1GiB", "op": "copy", "k": 0,
                      "gbs": round(2 * a1.numel() * 8 / (min(ts) * 1e-3) / 1e9, 1)}))
    del a1, b1
    tag = f"{os.environ.get('BK_SPMM_KERNEL', 'pipe')}/vec{os.environ.get('BK_SPMM_VEC', '8')}"
    for k in [int(x) for x in args.ks.split(",")]:
        X = synth.multivector(n, k, 3, device=dev)
        Y = torch.empty_like(X)
        C = synth.small_dense(k, k, 6, device=dev)
        G = torch.empty(k, k, dtype=torch.float64, device=dev)
        Cw = synth.window_coupling(k, 2).to(dev) if k % 2 == 0 else C   # SDIRK2 window coupling (sparse)
        ops = {"spmm": (lambda: bk.bspmm_apply(ctx, M, X, Y), pm.spmm_bytes(n, nnz, k)),
               "spmm_C": (lambda: bk.bspmm_apply(ctx, M, X, Y, C=C), pm.spmm_bytes(n, nnz, k)),
               "spmm_Cw": (lambda: bk.bspmm_apply(ctx, M, X, Y, C=Cw), pm.spmm_bytes(n, nnz, k)),
               "gram": (lambda: bk.block_gram(ctx, X, Y, G), pm.gram_bytes(n, k, k)),
               "update": (lambda: bk.block_update(ctx, Y, X, C, a=1.0, s=1e-3), pm.update_bytes(n, k, k))}
        for op in args.ops.split(","):
            fn, by = ops[op]
            ts = []
            for _ in range(args.reps):
                do_flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(args.batch):
                    fn()
                b.record(st)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts[1:]) / args.batch
            gbs = by / (ms * 1e-3) / 1e9
            print(json.dumps({"tag": tag, "cfg": args.cfg, "op": op, "k": k, "us": round(ms * 1e3, 2),
                              "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}))


if __name__ == "__main__":
    main()
