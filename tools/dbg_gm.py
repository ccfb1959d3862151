import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, synth, paper_2504_02117_b200 as m
c = m.Context(0)
A = synth.convdiff2d(256)
M = m.Matrix.from_csr(c, A)
for k in (4, 8, 12, 16):
    B = synth.multivector(A.n_rows, k, 2).cuda()
    X = torch.zeros_like(B)
    st, r = m.block_krylov_solve(c, M, B, X, method="gmres", rtol=1e-8, max_iters=400, restart=20, x0_is_zero=True)
    print(json.dumps({"bm": os.environ.get("BK_GMRES_BM"), "k": k, "st": st, "its": r["iterations"],
                      "relres": float(max(r["relres"])), "true": float(max(r["true_relres"]))}), flush=True)
