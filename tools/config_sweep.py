"""Per-config measurements (BASELINE.json configs c3, c4, c5): apply / Gram /
update GB/s at each config's k (L2 flushed before every launch, median of reps) and the
per-iteration time of the block solvers (slope over two iteration counts).

    python tools/config_sweep.py [--cfgs c3,c4,c5] [--reps 5] [--solve-iters 3,6]
Prints one JSON line per config.  Inputs are the seeded synthetic generators (synth).
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
from paper_2504_02117_b200 import perfmodel as pm  # noqa: E402
import synth  # noqa: E402

KS = {"c2": [8, 16, 32], "c3": [12], "c4": [16], "c5": [8, 16, 32]}
SOLVERS = {"c2": ["bicgstab", "cg"], "c3": ["gmres", "bicgstab"], "c4": ["cg", "bicgstab"], "c5": ["cg"]}


def peak():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, flush, reps):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfgs", default="c3,c4,c5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--solve-iters", default="3,6")
    args = ap.parse_args()
    P = peak()
    ctx = bk.Context(0)
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    it0, it1 = [int(x) for x in args.solve_iters.split(",")]
    for cfg in args.cfgs.split(","):
        t0 = time.time()
        A = synth.make_matrix(cfg, device=dev)
        torch.cuda.synchronize()
        t_gen = time.time() - t0
        t0 = time.time()
        M = bk.Matrix.from_csr(ctx, A)
        t_setup = time.time() - t0
        info = M.info()
        n, nnz = info["n_local"], info["nnz"]
        del A
        out = {"cfg": cfg, "n": n, "nnz": nnz, "n_bands": info["n_bands"], "gen_s": round(t_gen, 2),
               "setup_s": round(t_setup, 2), "peak_gbs": P, "kernels": {}, "solve_ms_per_iter": {}}
        for k in KS[cfg]:
            X = synth.multivector(n, k, 3, device=dev)
            Y = torch.empty_like(X)
            Pm = synth.multivector(n, k, 5, device=dev)
            C = synth.small_dense(k, k, 6, device=dev)
            G = torch.empty(k, k, dtype=torch.float64, device=dev)
            for name, fn, by in (("spmm", lambda: bk.bspmm_apply(ctx, M, X, Y), pm.spmm_bytes(n, nnz, k)),
                                 ("gram", lambda: bk.block_gram(ctx, X, Y, G), pm.gram_bytes(n, k, k)),
                                 ("update", lambda: bk.block_update(ctx, Pm, X, C, a=1.0, s=1e-3),
                                  pm.update_bytes(n, k, k))):
                ms = timed(fn, flush, args.reps)
                gbs = by / (ms * 1e-3) / 1e9
                out["kernels"][f"{name}_k{k}"] = {"us": round(ms * 1e3, 1), "gbs": round(gbs, 1),
                                                  "frac": round(gbs / P, 4)}
            del X, Y, Pm
        k = KS[cfg][-1] if cfg != "c5" else 16
        B = synth.multivector(n, k, 2, device=dev)
        Xs = torch.zeros_like(B)
        for meth in SOLVERS[cfg]:
            ms = {}
            for its in (it0, it1):
                def run(its=its):
                    bk.block_krylov_solve(ctx, M, B, Xs, method=meth, rtol=0.0, max_iters=its, x0_is_zero=True,
                                          check_every=its, restart=max(it1, 2))
                run()
                ms[its] = timed(run, flush, 2)
            slope = (ms[it1] - ms[it0]) / (it1 - it0)
            entry = {"k": k, "ms_per_iter": round(slope, 4)}
            if meth == "bicgstab":
                by = pm.bicgstab_iter_bytes(n, nnz, k)
                entry.update(gbs=round(by / (slope * 1e-3) / 1e9, 1), frac=round(by / (slope * 1e-3) / 1e9 / P, 4))
            elif meth == "cg":
                by = pm.cg_iter_bytes(n, nnz, k)
                entry.update(gbs=round(by / (slope * 1e-3) / 1e9, 1), frac=round(by / (slope * 1e-3) / 1e9 / P, 4))
            out["solve_ms_per_iter"][meth] = entry
        del B, Xs
        M.close()
        torch.cuda.empty_cache()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
