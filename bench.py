#!/usr/bin/env python
"""Benchmark of the block-Krylov hot path (BASELINE.json metric: block-SpMM GB/s & GFLOP/s,
fraction of HBM peak, vs k; block-Krylov solve time) on B200.

One STEP = one pass of the whole hot path over the c2 workload (BASELINE.json
configs[1]: 2-D convection-diffusion, 1024 x 1024 cells, 5-point CSR fp64):
    for k in (16, 8, 4, 2, 1):  bspmm_apply (Y = A X_k), block_gram (X_k^T Y_k),
                                block_update (P_k += 1e-3 X_k C_k)
    + block_krylov_solve: 5 fixed block-BiCGStab iterations at k = 16
(a1 apply, a3 Gram, a4 small dense, a5 update, a6 solver; a2 halo when N > 1).
`value` = algorithmic bytes of the step / device time of the step (GB/s).
L2 (126 MB) is flushed by a 512 MiB write before every timed step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): weak scaling, a 1024 x (1024 N) grid row-partitioned across
ranks (z/y-slabs), NCCL halo exchange inside bspmm_apply, NCCL allreduce of the
Gram matrices; time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KS = (1, 2, 4, 8, 16)
# launch order inside a step: widest first, so the host's launch queue is ahead of the device by the
# time the 6-25 us kernels of k <= 4 run (right after the step's opening synchronize the host,
# ~15 us per call through ctypes, would otherwise be what the device waits on)
STEP_KS = tuple(sorted(KS, reverse=True))
SOLVE_K = 16
SOLVE_ITERS = 5
UPD_SCALE = 1e-3
NX = 1024


def load_perfmodel():
    """perfmodel.py (host-only byte model) loaded by path: importing the package would map
    libbk.so, which the reference (oracle) arm must not load."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bk_perfmodel", os.path.join(ROOT, "paper_2504_02117_b200",
                                                                                 "perfmodel.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def step_bytes(pm, n, nnz, ks=KS, solve_k=SOLVE_K, solve_iters=SOLVE_ITERS, n_ghost_rows=0, fused_apply=True):
    """Algorithmic bytes / flops of one step (perfmodel.py)."""
    b = f = 0
    parts = {}
    for k in ks:
        sb = pm.spmm_bytes(n, nnz, k, n_ghost=n_ghost_rows)
        gb = pm.gram_bytes(n, k, k)
        ub = pm.update_bytes(n, k, k)
        parts[k] = dict(spmm=sb, gram=gb, update=ub, spmm_flops=pm.spmm_flops(nnz, k),
                        gram_flops=pm.gram_flops(n, k, k), update_flops=pm.update_flops(n, k, k))
        b += sb + gb + ub
        f += parts[k]["spmm_flops"] + parts[k]["gram_flops"] + parts[k]["update_flops"]
    # solve: x0 = 0 -> R = B (copy), ||R||, Rt aliases B (no copy), P = R, iterations, final
    # true residual -- only the passes solve.cpp enqueues (the library reports the same count as
    # bk_solve_report.alg_bytes; run_ours checks the two agree)
    sb = pm.bicgstab_solve_bytes(n, nnz, solve_k, solve_iters, fused_apply=fused_apply)
    parts["solve"] = dict(bytes=sb)
    b += sb
    return b, f, parts


# ------------------------------------------------------------------ clocks
class Clocks:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
            self._wait_lines(1, 5.0)       # sampler running before the timed region starts
            self.n0 = self._lines()
        except Exception:
            self.proc = None
        return self

    def _lines(self):
        try:
            return sum(1 for ln in open(self.path) if ln.strip())
        except Exception:
            return 0

    def _wait_lines(self, n, timeout):
        t0 = time.time()
        while self._lines() < n and time.time() - t0 < timeout:
            time.sleep(0.01)

    def __exit__(self, *a):
        if self.proc:
            self._wait_lines(self.n0 + 1, 1.0)   # at least one sample taken during the region
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self, device_index=0):
        try:
            rows = [ln.split(",") for ln in open(self.path) if ln.strip()]
        except Exception:
            return None
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 9 and r[0].strip() == str(device_index)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_02117_b200 as bk
    import synth
    pm = load_perfmodel()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if rank == 0:
            print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = bk.Context(local)
    if world > 1:
        uid = bk.Context.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, 0)
        ctx.set_comm(bytes(t.cpu().tolist()), world, rank)

    # ---- workload: c2 (N = 1) or the weak-scaled 1024 x 1024N grid, this rank's row slab
    ny = NX * world
    A_full = synth.convdiff2d(NX, ny=ny, device=dev)
    n_glob = A_full.n_rows
    r0, r1 = rank * n_glob // world, (rank + 1) * n_glob // world
    A = A_full.rows(r0, r1) if world > 1 else A_full
    del A_full
    M = bk.Matrix(ctx, A.row_ptr, A.col, A.val, n_global=n_glob, row_begin=r0, n_local=r1 - r0)
    info = M.info()
    n, nnz = info["n_local"], info["nnz"]
    X = {k: synth.multivector(n, k, synth.SEEDS["X"], row_begin=r0, n_global=n_glob, device=dev) for k in KS}
    Y = {k: torch.empty(n, k, dtype=torch.float64, device=dev) for k in KS}
    P = {k: synth.multivector(n, k, synth.SEEDS["P"], row_begin=r0, n_global=n_glob, device=dev) for k in KS}
    C = {k: synth.small_dense(k, k, synth.SEEDS["C"], device=dev) for k in KS}
    G = {k: torch.empty(k, k, dtype=torch.float64, device=dev) for k in KS}
    B = synth.multivector(n, SOLVE_K, synth.SEEDS["B"], row_begin=r0, n_global=n_glob, device=dev)
    Xs = torch.zeros(n, SOLVE_K, dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    flush_sink = torch.empty((), dtype=torch.float64, device=dev)

    def flush_l2():
        # write a buffer 4x the L2, then read it: L2 holds clean lines of the flush buffer, so
        # the next kernel neither hits its inputs nor pays write-backs of the flush (the
        # isolated-kernel harness tools/sweep.py does the same)
        flush.fill_(1.0)
        torch.sum(flush, dim=0, out=flush_sink)

    stream = torch.cuda.current_stream(dev)
    allred = world > 1

    solve_cls = []   # per timed step: the solver's per-kernel-class event times (opts.timing)

    def one_step(ev=None, timed=False):
        # ev[key] = (start, end); start is the previous key's end event (recorded already)
        for k in STEP_KS:
            bk.bspmm_apply(ctx, M, X[k], Y[k])
            if ev is not None:
                ev[("spmm", k)][1].record(stream)
            bk.block_gram(ctx, X[k], Y[k], G[k], allreduce=allred)
            if ev is not None:
                ev[("gram", k)][1].record(stream)
            bk.block_update(ctx, P[k], X[k], C[k], a=1.0, s=UPD_SCALE)
            if ev is not None:
                ev[("update", k)][1].record(stream)
        st, rep = bk.block_krylov_solve(ctx, M, B, Xs, method="bicgstab", rtol=0.0, max_iters=SOLVE_ITERS,
                                        x0_is_zero=True, check_every=SOLVE_ITERS, timing=timed)
        if ev is not None:
            ev[("solve", SOLVE_K)][1].record(stream)
        if timed:
            solve_cls.append((rep["t_class_ms"], rep["n_class"]))
        return rep

    # warm-up
    rep_w = None
    for _ in range(args.warmup):
        rep_w = one_step()
    torch.cuda.synchronize()
    solve_bytes_lib = rep_w["alg_bytes"] if rep_w else None
    if getattr(args, "profile_step", False):
        # one step between cudaProfilerStart/Stop, for `ncu --profile-from-start off`
        flush_l2()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        one_step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return

    keys = [(c, k) for k in STEP_KS for c in ("spmm", "gram", "update")] + [("solve", SOLVE_K)]
    durs = {kk: [] for kk in keys}
    step_ms = []
    launches0 = bk.kernel_launch_count()
    clocks = Clocks(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else ".",
                                 f".bench_clocks_{rank}.csv"))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with clocks:
        for step in range(args.steps):
            flush_l2()                                         # L2 flush (outside the step timing)
            ev = {kk: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for kk in keys}
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            # chain: each kernel's start event is the previous kernel's end event
            prev = e0
            one_step_ev = {}
            for kk in keys:
                one_step_ev[kk] = (prev, ev[kk][1])
                prev = ev[kk][1]
            # the solver's per-kernel events (opts.timing) only in the last timed step:
            # they add gaps between kernels, so the other steps run without them
            # per-kernel events only in the last (up to) three timed steps: every record between two
            # kernels costs host time and a device-side gap
            inst = step >= args.steps - 3
            one_step(one_step_ev if inst else None, timed=(step == args.steps - 1))
            if not inst:
                prev.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(prev))
            if inst:
                for kk in keys:
                    a, b = one_step_ev[kk]
                    durs[kk].append(a.elapsed_time(b))
        torch.cuda.synchronize()
    launches = bk.kernel_launch_count() - launches0
    if world > 1:
        dist.barrier()
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    n_ghost = info["n_ghost"]
    # one rank: the fused BiCGStab takes its reductions in the applies' epilogues (2-D band plan)
    bytes_rank, flops_rank, parts = step_bytes(pm, n, nnz, n_ghost_rows=n_ghost, fused_apply=(world == 1))
    if solve_bytes_lib is not None and solve_bytes_lib != parts["solve"]["bytes"]:
        raise RuntimeError(f"byte model of the solve ({parts['solve']['bytes']}) != the solver's own count "
                           f"({solve_bytes_lib})")
    bytes_all = bytes_rank * world
    value = bytes_all / (ms_per_step * 1e-3) / 1e9

    # ---- per-kernel (mean device time inside the timed region)
    peak, peak_src = peaks()
    per = {}
    for (c, k) in keys:
        mean_ms = sum(durs[(c, k)]) / len(durs[(c, k)])
        if c == "solve":
            by = parts["solve"]["bytes"]
            per[f"solve_k{k}"] = dict(ms=mean_ms, gbs=by / (mean_ms * 1e-3) / 1e9,
                                      ms_per_iter=mean_ms / SOLVE_ITERS)
        else:
            by = parts[k][c]
            fl = parts[k][c + "_flops"]
            per[f"{c}_k{k}"] = dict(ms=mean_ms, gbs=by / (mean_ms * 1e-3) / 1e9,
                                    gflops=fl / (mean_ms * 1e-3) / 1e9, frac=by / (mean_ms * 1e-3) / 1e9 / peak)
    # ---- dominant kernel: largest share of the step.  Kernels inside the solve are timed by
    # the library's CUDA events on the ctx stream (opts.timing); the k = 16 apply runs both
    # as the microbenchmark call and inside the solve (same kernel: times and launches merged).
    v16 = 8 * n * SOLVE_K
    cls_ms = {c: sum(t[c] for t, _ in solve_cls) / len(solve_cls) for c in solve_cls[0][0]}
    cls_n = {c: sum(m[c] for _, m in solve_cls) / len(solve_cls) for c in solve_cls[0][1]}
    sb16 = pm.spmm_bytes(n, nnz, SOLVE_K, n_ghost=info["n_ghost"])
    kern = {
        "bcg_tail_k16": dict(ms=cls_ms["fused_tail"], n=cls_n["fused_tail"], bytes=8 * v16),
        "fused_gram_k16": dict(ms=cls_ms["fused_gram"], n=cls_n["fused_gram"], bytes=3 * v16),
        "fused_dots_k16": dict(ms=cls_ms["fused_dots"], n=cls_n["fused_dots"], bytes=3 * v16),
        "spmm_k16": dict(ms=cls_ms["spmm"] + per["spmm_k16"]["ms"], n=cls_n["spmm"] + 1, bytes=sb16),
        # the applies with a reduction in their epilogue (two kernels, bspmm_win_kernel<.., RED>):
        # V = A P with Rt^T [V R] (+ Rt, R read) and T = A S with Rt^T T, <T,S>, <T,T> (+ Rt)
        "fused_apply_gram_k16": dict(ms=cls_ms.get("fused_apply", 0.0), n=cls_n.get("fused_apply", 0),
                                     bytes=sb16 + 2 * v16),
        "fused_apply_dots_k16": dict(ms=cls_ms.get("fused_apply_dots", 0.0), n=cls_n.get("fused_apply_dots", 0),
                                     bytes=sb16 + v16),
    }
    for kk, v in per.items():
        if not kk.startswith("solve") and kk not in kern:
            c, k = kk.split("_k")
            kern[kk] = dict(ms=v["ms"], n=1, bytes=parts[int(k)][c])
    shares = {kk: round(v["ms"] / ms_per_step, 4) for kk, v in kern.items() if v["n"] > 0}
    dom = max((kk for kk in kern if kern[kk]["n"] > 0), key=lambda kk: kern[kk]["ms"])
    dk = kern[dom]
    avg_ms = dk["ms"] / dk["n"]
    achieved = dk["bytes"] / (avg_ms * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "alg_bytes": dk["bytes"], "peak_source": peak_src,
                "launches_per_step": dk["n"], "avg_launch_ms": avg_ms, "share_of_step": dk["ms"] / ms_per_step,
                "shares": dict(sorted(shares.items(), key=lambda x: -x[1])[:8])}

    # ---- isolated k sweep (flush before every kernel; adds k = 32), outside the timed region
    sweep = {}
    if not args.no_sweep:
        for k in (1, 2, 4, 8, 12, 16, 20, 24, 32):   # (12 / 20 / 24: the lane-exact gather instantiations)
            Xk = X[k] if k in X else synth.multivector(n, k, synth.SEEDS["X"], row_begin=r0, n_global=n_glob, device=dev)
            Yk = torch.empty(n, k, dtype=torch.float64, device=dev)
            Pk = P[k] if k in P else synth.multivector(n, k, synth.SEEDS["P"], device=dev)
            Ck = C[k] if k in C else synth.small_dense(k, k, synth.SEEDS["C"], device=dev)
            Gk = torch.empty(k, k, dtype=torch.float64, device=dev)
            row = {}
            for name, fn, by, fl in (
                    ("spmm", lambda: bk.bspmm_apply(ctx, M, Xk, Yk), pm.spmm_bytes(n, nnz, k, n_ghost=n_ghost),
                     pm.spmm_flops(nnz, k)),
                    ("spmm_C", lambda: bk.bspmm_apply(ctx, M, Xk, Yk, C=Ck), pm.spmm_bytes(n, nnz, k, n_ghost=n_ghost),
                     pm.spmm_flops(nnz, k, n, coupled=True)),
                    ("gram", lambda: bk.block_gram(ctx, Xk, Yk, Gk, allreduce=allred), pm.gram_bytes(n, k, k),
                     pm.gram_flops(n, k, k)),
                    ("update", lambda: bk.block_update(ctx, Pk, Xk, Ck, a=1.0, s=UPD_SCALE), pm.update_bytes(n, k, k),
                     pm.update_flops(n, k, k))):
                ts = []
                for _ in range(7):
                    flush_l2()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    fn()
                    b.record(stream)
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                ms = statistics.median(ts[1:])
                row[name] = dict(us=round(ms * 1e3, 2), gbs=round(by / (ms * 1e-3) / 1e9, 1),
                                 gflops=round(fl / (ms * 1e-3) / 1e9, 1), frac=round(by / (ms * 1e-3) / 1e9 / peak, 4))
            sweep[k] = row

    # ---- the other BASELINE configs (c3, c4, c5), outside the timed region: apply / Gram /
    # update GB/s at each config's k and block-solver time per iteration (tools/config_sweep.py)
    configs = None
    if world == 1 and not args.no_sweep and not args.no_configs:
        try:
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "config_sweep.py"), "--cfgs", "c3,c4,c5"],
                               capture_output=True, text=True, timeout=900)
            configs = {}
            for ln in r.stdout.splitlines():
                try:
                    d = json.loads(ln)
                    configs[d.pop("cfg")] = d
                except ValueError:
                    pass
            if r.returncode != 0:
                configs["error"] = r.stderr[-400:]
        except Exception as e:   # never fail the bench line on the side measurements
            configs = {"error": str(e)[:400]}

    # ---- solve time (full solves, outside the timed region): c1 block GMRES k=4 to 1e-10
    solve_report = None
    if world == 1 and not args.no_sweep:
        A1 = synth.make_matrix("c1")
        M1 = bk.Matrix.from_csr(ctx, A1)
        B1 = synth.multivector(A1.n_rows, 4, synth.SEEDS["B"], device=dev)
        X1 = torch.zeros_like(B1)
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st, rep = bk.block_krylov_solve(ctx, M1, B1, X1, method="gmres", restart=100, rtol=1e-10, x0_is_zero=True)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        solve_report = {"c1_gmres_k4_ms": statistics.median(ts), "iterations": rep["iterations"],
                        "converged": rep["converged"], "max_true_relres": float(max(rep["true_relres"]))}
        # block CG (symmetric c1 variant) and block BiCGStab to 1e-10, iterations replayed from a
        # CUDA graph (bk_solve_opts.use_graphs), convergence polled every 8 iterations
        for name, cfg1, meth in (("c1s_cg_k4", "c1s", "cg"), ("c1_bicgstab_k4", "c1", "bicgstab")):
            A1 = synth.make_matrix(cfg1)
            M1 = bk.Matrix.from_csr(ctx, A1)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                st, rep = bk.block_krylov_solve(ctx, M1, B1, X1, method=meth, rtol=1e-10, x0_is_zero=True,
                                                use_graphs=True, check_every=8)
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            solve_report[name + "_graphs_ms"] = statistics.median(ts)
            solve_report[name + "_iterations"] = rep["iterations"]
            solve_report[name + "_max_true_relres"] = float(max(rep["true_relres"]))

    if world == 1 and not args.no_sweep and not args.no_solves and solve_report is not None:
        try:
            solve_report.update(solve_benchmarks(bk, ctx, dev))
        except Exception as e:   # never fail the bench line on the side measurement
            solve_report["error"] = str(e)[:400]

    # ---- e2e: same step through the C ABI with pinned HOST buffers (H2D/D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        hX = {k: X[k].cpu().pin_memory() for k in KS}
        hY = {k: torch.empty(n, k, dtype=torch.float64).pin_memory() for k in KS}
        hP = {k: P[k].cpu().pin_memory() for k in KS}
        hC = {k: C[k].cpu().pin_memory() for k in KS}
        hG = {k: torch.empty(k, k, dtype=torch.float64).pin_memory() for k in KS}
        hB = B.cpu().pin_memory()
        hXs = torch.zeros(n, SOLVE_K, dtype=torch.float64).pin_memory()

        def host_step():
            for k in KS:
                bk.bspmm_apply(ctx, M, hX[k], hY[k])
                bk.block_gram(ctx, hX[k], hY[k], hG[k], allreduce=allred)
                bk.block_update(ctx, hP[k], hX[k], hC[k], a=1.0, s=UPD_SCALE)
            bk.block_krylov_solve(ctx, M, hB, hXs, method="bicgstab", rtol=0.0, max_iters=SOLVE_ITERS,
                                  x0_is_zero=True, check_every=SOLVE_ITERS)

        host_step()
        e_steps = max(3, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ts = []
        for _ in range(e_steps):
            flush_l2()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            host_step()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        e_ms = sum(ts) / len(ts)
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        h2d = sum(8 * n * k + 16 * n * k + (16 * n * k + 8 * k * k) for k in KS) + 8 * n * SOLVE_K
        d2h = sum(8 * n * k + 8 * k * k + 8 * n * k for k in KS) + 8 * n * SOLVE_K
        e2e = {"value": bytes_all / (e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "note": "same step via the C ABI with pinned host X/Y/P/C/G/B buffers; host wall clock"}

    # ---- strong scaling on the largest grid (N > 1, or --strong-c5 at N = 1)
    strong = None
    if (world > 1 and not args.no_strong) or args.strong_c5:
        try:
            strong = strong_c5(bk, ctx, world, rank, dev)
        except Exception as e:   # never fail the bench line on the side measurement
            strong = {"error": str(e)[:400]}

    # ---- CPU oracle baseline (rank 0, N = 1): bounded sample of the same step
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(rows=65536, reps=args.cpu_reps)

    if rank == 0:
        cs = clocks.summary(local)
        line = {
            "metric": "block-SpMM GB/s & GFLOP/s (fraction of HBM peak) vs k; block-Krylov solve time",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded SplitMix64 inputs; FV matrices assembled on device)",
            "config": {"workload": "c2" if world == 1 else f"c2-weak-{world}",
                       "grid": f"{NX}x{ny}", "rows_per_gpu": n, "nnz_per_gpu": nnz, "ks": list(KS),
                       "solve": f"block BiCGStab k={SOLVE_K}, {SOLVE_ITERS} iterations",
                       "step_alg_bytes_per_gpu": bytes_rank, "step_flops_per_gpu": flops_rank,
                       "solve_alg_bytes_reported_by_library": solve_bytes_lib,
                       "l2": "flushed (512 MiB write, then read: clean L2) before every timed step and every swept kernel",
                       "parallelism": "single GPU" if world == 1 else f"row partition x{world}, NCCL halo + allreduce"},
            "gpu_launches": launches,
            "roofline": roofline,
            "per_kernel": per,
            "sweep": sweep,
            "solve": solve_report,
            "configs": configs,
            "e2e": e2e,
            "strong_scaling_c5": strong,
            "cpu_baseline": cpu,
            "clocks": cs,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------ full solves (the metric's "block-Krylov solve time")
BCG_RHS = 128
BCG_KS = (1, 2, 4, 8, 16, 32)


def solve_benchmarks(bk, ctx, dev, bcg_grid=96):
    """BASELINE.json's solve-time half of the metric, outside the timed region:
    * c3 (BJ configs[2]): block GMRES(64), k = 12, rtol 1e-10, X0 = 0 -- time, block iterations,
      recomputed true residual;
    * the analog of the paper's Block-CG benchmark (Fig. bcgbenchmark): 128
      right-hand sides solved k at a time (k = 1, 2, 4, 8, 16, 32) to a defect reduction of 1e-8 for
      all of them, on the Richards-type stiffness matrix (the c4 recipe, R20/R21) at bcg_grid^3, block
      CG preconditioned by the Chebyshev polynomial (R28; the paper uses AMG, out of scope): total time
      and block iterations per chunk."""
    import torch
    import synth
    out = {}
    A = synth.make_matrix("c3", device=dev)
    M = bk.Matrix.from_csr(ctx, A)
    k = 12
    B = synth.multivector(A.n_rows, k, synth.SEEDS["B"], device=dev)
    X = torch.zeros_like(B)
    bk.block_krylov_solve(ctx, M, B, X, method="gmres", restart=64, rtol=1e-10, max_iters=2, x0_is_zero=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    st, rep = bk.block_krylov_solve(ctx, M, B, X, method="gmres", restart=64, rtol=1e-10, max_iters=2000,
                                    x0_is_zero=True, check_every=4)
    b.record()
    torch.cuda.synchronize()
    out["c3_gmres64_k12"] = {"ms": a.elapsed_time(b), "block_iterations": rep["iterations"],
                             "converged": rep["converged"], "max_true_relres": float(max(rep["true_relres"])),
                             "rtol": 1e-10}
    del M, A, B, X
    torch.cuda.empty_cache()
    n3 = bcg_grid
    A = synth.richards3d(n3, n3, n3, device=dev)
    M = bk.Matrix.from_csr(ctx, A)
    Ball = synth.multivector(A.n_rows, BCG_RHS, synth.SEEDS["B"], device=dev)
    rows = {}
    for k in BCG_KS:
        Bk = [Ball[:, c:c + k].contiguous() for c in range(0, BCG_RHS, k)]
        Xk = torch.zeros_like(Bk[0])
        bk.block_krylov_solve(ctx, M, Bk[0], Xk, method="cg", precond="chebyshev", cheb_steps=4, rtol=1e-8,
                              max_iters=2, x0_is_zero=True)
        its, worst = [], 0.0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for Bc in Bk:
            st, rep = bk.block_krylov_solve(ctx, M, Bc, Xk, method="cg", precond="chebyshev", cheb_steps=4,
                                            rtol=1e-8, max_iters=5000, x0_is_zero=True, check_every=8)
            its.append(rep["iterations"])
            worst = max(worst, float(max(rep["true_relres"])))
        b.record()
        torch.cuda.synchronize()
        rows[k] = {"ms": a.elapsed_time(b), "chunks": len(Bk), "iterations_per_chunk": sorted(set(its)),
                   "max_true_relres": worst}
    out["bcg128_richards"] = {"grid": f"{n3}^3", "rows": A.n_rows, "rhs": BCG_RHS, "rtol": 1e-8,
                              "precond": "chebyshev(4 steps, Gershgorin interval)", "by_k": rows,
                              "fastest_k": min(rows, key=lambda kk: rows[kk]["ms"])}
    return out


# ------------------------------------------------------------------ strong scaling on c5 (north star E(N))
STRONG_KS = (8, 16, 32)
STRONG_CG_K, STRONG_CG_ITERS = 16, 20


def strong_c5(bk, ctx, world, rank, dev, reps=3):
    """parallel efficiency E(N) = T(1) / (N T(N)) on the largest grid (c5,
    512 x 512 x 256, 67.1 M rows) for the block apply at k = 8 / 16 / 32 and for 20 fixed block-CG
    iterations at k = 16, the matrix row-partitioned into z-slabs (NCCL halo + Gram allreduce).
    T(1) is measured in the same run on rank 0's GPU alone (a single-rank context), then T(N) on
    all ranks (CUDA events, max over ranks)."""
    import torch
    import torch.distributed as dist
    import synth
    A = synth.make_matrix("c5", device=dev)
    n = A.n_rows
    plane = 512 * 512
    nz = n // plane
    rb = [(nz * r // world) * plane for r in range(world + 1)]
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def run(c, M, r0, r1, allred):
        nl = r1 - r0
        big_x = torch.empty(nl * max(STRONG_KS), dtype=torch.float64, device=dev)
        big_y = torch.empty_like(big_x)
        st = torch.cuda.current_stream(dev)
        out = {}
        for k in STRONG_KS:
            X = big_x[:nl * k].view(nl, k)
            X.copy_(synth.multivector(nl, k, synth.SEEDS["X"], row_begin=r0, n_global=n, device=dev))
            Y = big_y[:nl * k].view(nl, k)
            ts = []
            for _ in range(reps + 1):
                flush.fill_(1.0)
                if allred:
                    dist.barrier()
                torch.cuda.synchronize(dev)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                bk.bspmm_apply(c, M, X, Y)
                b.record(st)
                torch.cuda.synchronize(dev)
                ts.append(a.elapsed_time(b))
            out[f"spmm_k{k}"] = min(ts[1:])
        k = STRONG_CG_K
        B = big_x[:nl * k].view(nl, k)
        B.copy_(synth.multivector(nl, k, synth.SEEDS["B"], row_begin=r0, n_global=n, device=dev))
        Xs = big_y[:nl * k].view(nl, k)
        ts = []
        for _ in range(2):
            if allred:
                dist.barrier()
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            bk.block_krylov_solve(c, M, B, Xs, method="cg", rtol=0.0, max_iters=STRONG_CG_ITERS, x0_is_zero=True,
                                  check_every=STRONG_CG_ITERS)
            b.record(st)
            torch.cuda.synchronize(dev)
            ts.append(a.elapsed_time(b))
        out[f"cg_k{k}_{STRONG_CG_ITERS}it"] = ts[-1]
        del big_x, big_y
        torch.cuda.empty_cache()
        if allred:   # max over ranks
            t = torch.tensor([out[kk] for kk in sorted(out)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out = dict(zip(sorted(out), t.tolist()))
        return out

    t1 = None
    if rank == 0:
        c1 = bk.Context(dev.index)
        M1 = bk.Matrix(c1, A.row_ptr, A.col, A.val)
        t1 = run(c1, M1, 0, n, False)
        M1.close()
        c1.close()
        torch.cuda.empty_cache()
    tn = None
    if world > 1:
        dist.barrier()
        S = A.rows(rb[rank], rb[rank + 1])
        del A
        torch.cuda.empty_cache()
        M = bk.Matrix(ctx, S.row_ptr, S.col, S.val, n_global=n, row_begin=rb[rank], n_local=rb[rank + 1] - rb[rank])
        del S
        tn = run(ctx, M, rb[rank], rb[rank + 1], True)
        M.close()
    if rank != 0:
        return None
    res = {"workload": "c5 (512x512x256, 7-point Richards-type, fp64), z-slab row partition", "n_gpus": world,
           "T1_ms": t1, "TN_ms": tn, "reps": reps,
           "note": "apply: min of reps after one warm-up, L2 flushed before each; CG: 20 fixed iterations "
                   "(second of two runs), setup outside the timed region"}
    if tn:
        res["efficiency"] = {kk: t1[kk] / (world * tn[kk]) for kk in t1}
    return res


# ------------------------------------------------------------------ oracle (CPU) arm
def _oracle_sample(rows):
    """Leading `rows` x `rows` principal block of c2 (a valid smaller instance of the same operator)."""
    import synth
    A = synth.make_matrix("c2")
    rows = min(rows, A.n_rows)
    S = A.rows(0, rows)
    keep = S.col < rows
    counts = torch_counts(S.row_ptr, keep)
    import torch
    rp = torch.zeros(rows + 1, dtype=torch.int64)
    rp[1:] = torch.cumsum(counts, 0)
    return synth.Csr(rows, rows, rp.to(torch.int32), S.col[keep].contiguous(), S.val[keep].contiguous(), "c2-sample")


def torch_counts(row_ptr, keep):
    import torch
    rp = row_ptr.to(torch.int64)
    cs = torch.zeros(len(keep) + 1, dtype=torch.int64)
    cs[1:] = torch.cumsum(keep.to(torch.int64), 0)
    return cs[rp[1:]] - cs[rp[:-1]]


def oracle_step_fn(rows):
    import numpy as np
    import oracle
    import synth
    A = _oracle_sample(rows)
    Ao = oracle.CsrNp.of(A)
    n = A.n_rows
    X = {k: synth.multivector(n, k, synth.SEEDS["X"]).numpy() for k in KS}
    P = {k: synth.multivector(n, k, synth.SEEDS["P"]).numpy() for k in KS}
    C = {k: synth.small_dense(k, k, synth.SEEDS["C"]).numpy() for k in KS}
    B = synth.multivector(n, SOLVE_K, synth.SEEDS["B"]).numpy()

    def step():
        for k in KS:
            Y = oracle.spmm(Ao, X[k])
            oracle.gram(X[k], Y)
            P[k] = oracle.update(P[k], X[k], C[k], 1.0, UPD_SCALE)
        oracle.block_bicgstab(Ao, B, rtol=0.0, max_iters=SOLVE_ITERS)
        return np.zeros(1)

    return step, n, A.nnz


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_timing(rows, procs, reps, warmup=0):
    """Run in a fresh interpreter with every BLAS / OpenMP pool at one thread (bench.py
    --oracle-timing): build the oracle step on the leading `rows`-row principal block of c2, fork
    `procs` workers that run it concurrently (each worker one core: the oracle is plain
    single-threaded C + numpy), `warmup` + `reps` rounds separated by a barrier.  Returns the
    per-round wall time of the slowest worker (seconds) and the step's algorithmic bytes."""
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMEXPR_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-timing", str(rows), str(procs), str(reps),
                        str(warmup)], env=env, capture_output=True, text=True, timeout=3600)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-800:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def _oracle_timing_main(rows, procs, reps, warmup):
    import multiprocessing as mp
    step, n, nnz = oracle_step_fn(rows)
    pm = load_perfmodel()
    by, _, _ = step_bytes(pm, n, nnz)
    ctx = mp.get_context("fork")
    bar = ctx.Barrier(procs)
    q = ctx.Queue()

    def worker(i):
        ts = []
        for _ in range(warmup + reps):
            bar.wait()
            t0 = time.perf_counter()
            step()
            ts.append(time.perf_counter() - t0)
        q.put((i, ts[warmup:]))

    ps = [ctx.Process(target=worker, args=(i,)) for i in range(procs)]
    for p in ps:
        p.start()
    res = dict(q.get() for _ in ps)
    for p in ps:
        p.join()
    rounds = [max(res[i][j] for i in range(procs)) for j in range(reps)]
    print(json.dumps({"rows": n, "nnz": nnz, "bytes": by, "procs": procs, "round_s": rounds}))


def cpu_baseline(rows=65536, reps=1):
    """The oracle as it stands on the host: 1 core, and every core of the job's affinity mask
    (one independent oracle process per core on the same sample: the oracle is single
    threaded, so all-core throughput = cores x sample bytes / slowest process)."""
    cores = host_cores()
    one = oracle_timing(rows, 1, reps)
    t1 = statistics.median(one["round_s"])
    allc = oracle_timing(rows, cores, reps) if cores > 1 else one
    ta = statistics.median(allc["round_s"])
    by, n, nnz = one["bytes"], one["rows"], one["nnz"]
    return {"value": cores * by / ta / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "single_core": {"value": by / t1 / 1e9, "unit": "GB/s", "cores": 1, "s_per_step": t1},
            "all_cores": {"value": cores * by / ta / 1e9, "unit": "GB/s", "cores": cores, "s_per_step": ta},
            "sample": f"same step on the leading {n}-row principal block of c2 ({nnz} nnz), {reps} rep(s); "
                      f"all cores = {cores} concurrent single-threaded oracle processes (plain C, gcc -O2, + numpy "
                      f"solver, BLAS at 1 thread), 1 core = one such process"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    rows = 32768
    cores = host_cores()
    r = oracle_timing(rows, cores, args.steps, args.warmup)
    ms = statistics.mean(r["round_s"]) * 1e3
    n, nnz = r["rows"], r["nnz"]
    v = cores * r["bytes"] / (ms * 1e-3) / 1e9
    sample = (f"same step (bspmm/gram/update at k=1,2,4,8,16 + 5 block-BiCGStab its at k=16) on the leading "
              f"{n}-row principal block of c2 ({nnz} nnz), run by {cores} concurrent single-threaded oracle "
              f"processes (one per host core); step time = slowest process")
    print(json.dumps({
        "impl": "reference", "metric": "block-SpMM GB/s & GFLOP/s (fraction of HBM peak) vs k; block-Krylov solve time",
        "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "c2" if world == 1 else f"c2-weak-{world}", "sample_rows": n},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--profile-step", action="store_true", help="one step inside cudaProfilerStart/Stop (ncu --profile-from-start off)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the c3/c4/c5 side measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=1)
    ap.add_argument("--no-strong", action="store_true", help="N > 1: skip the c5 strong-scaling section")
    ap.add_argument("--no-solves", action="store_true", help="skip the full-solve benchmarks (c3 GMRES, 128-RHS CG)")
    ap.add_argument("--strong-c5", action="store_true", help="run the c5 strong-scaling section at N = 1 too")
    ap.add_argument("--oracle-timing", nargs=4, type=int, metavar=("ROWS", "PROCS", "REPS", "WARMUP"),
                    help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.oracle_timing:
        _oracle_timing_main(*args.oracle_timing)
        return
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
