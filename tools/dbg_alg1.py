import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2504_02117_b200 as bk, oracle, synth
ctx = bk.Context(0)
for tab, w, shape in [("sdirk3", 3, (6,5,4)), ("sdirk3", 2, (6,5,4)), ("sdirk2", 3, (6,5,4))]:
    nx, ny, nz = shape; tau, nst = 0.05, 3
    A = synth.SDIRK2 if tab == "sdirk2" else synth.SDIRK3
    y0, g = synth.dr_fields(nx, ny, nz, 1)
    P = oracle.DRProblem(nx, ny, nz, y0.numpy(), g.numpy(), tau)
    eps = 1e-12 * np.sqrt(P.N) * P.mass / P.tau
    ref, its_ref = oracle.algorithm1(P, A, nst, w, eps=eps)
    for meth in ("gmres", "bicgstab"):
        st, its, rep = bk.alg1_run(ctx, nx, ny, nz, tau, y0.cuda(), g.cuda(), A, nst, w, eps, max_newton=20,
                                   method=meth, restart=60, rtol=1e-14, max_iters=600)
        print(tab, w, meth, st, its, its_ref, rep, flush=True)
