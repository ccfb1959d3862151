"""Small but ring-wrapping invocations of every TMA / mbarrier ring kernel, for
`compute-sanitizer --tool racecheck|synccheck` (one tool per run).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
Every persistent kernel gets a grid of 2 x SMs CTAs, so a ring wraps only with more than
2 x SMs x (stages) tiles: the sizes below give several tiles per CTA.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402
import synth  # noqa: E402


def main():
    ctx = bk.Context(0)
    # windowed apply (2-D, 3 bands): k = 3 (odd: hand-copied last row), 8, 16, 32 (split map), coupled
    A2 = synth.convdiff2d(512, ny=301)
    M2 = bk.Matrix.from_csr(ctx, A2)
    for k in (3, 8, 16, 32):
        X = synth.multivector(A2.n_rows, k, 3, device="cuda")
        Y = torch.empty_like(X)
        bk.bspmm_apply(ctx, M2, X, Y)
        C = synth.small_dense(k, k, 6, device="cuda")
        bk.bspmm_apply(ctx, M2, X, Y, C=C, alpha=-1.0, beta=0.5)
    # gather (pipe) apply (3-D, 5 bands): k = 8, 12 (three-lane kernel), 16, 32, coupled 16
    A3 = synth.diffreact3d(48)
    M3 = bk.Matrix.from_csr(ctx, A3)
    for k in (8, 12, 16, 32):
        X = synth.multivector(A3.n_rows, k, 3, device="cuda")
        Y = torch.empty_like(X)
        bk.bspmm_apply(ctx, M3, X, Y)
        if k == 16:
            bk.bspmm_apply(ctx, M3, X, Y, C=synth.small_dense(k, k, 6, device="cuda"))
    # streaming Gram / update / coldot
    n = 200_000
    for k in (1, 4, 8, 12, 16):
        X = synth.multivector(n, k, 3, device="cuda")
        Y = synth.multivector(n, k, 4, device="cuda")
        G = torch.empty(k, k, dtype=torch.float64, device="cuda")
        bk.block_gram(ctx, X, Y, G)
        bk.block_update(ctx, Y, X, G, a=1.0, s=1e-3)
    # fused solvers (panel Gram + epilogues, BiCGStab / CG tails with the stage write-back)
    A = synth.convdiff2d(384)
    As = synth.convdiff2d(384, v=(0.0, 0.0))
    M, Ms = bk.Matrix.from_csr(ctx, A), bk.Matrix.from_csr(ctx, As)
    for k in (4, 8, 12, 16):
        B = synth.multivector(A.n_rows, k, 2, device="cuda")
        X = torch.zeros_like(B)
        bk.block_krylov_solve(ctx, M, B, X, method="bicgstab", rtol=1e-30, max_iters=3, x0_is_zero=True)
        bk.block_krylov_solve(ctx, Ms, B, X, method="cg", rtol=1e-30, max_iters=3, x0_is_zero=True)
        bk.block_krylov_solve(ctx, Ms, B, X, method="cg1", rtol=1e-30, max_iters=3, x0_is_zero=True)
    # in-place P update (out == P) through the streaming DMMA kernel and the flat kernel
    for k in (2, 8, 16):
        P = synth.multivector(n, k, 3, device="cuda")
        bk.block_update(ctx, P, P, synth.small_dense(k, k, 6, device="cuda"), a=1.0, s=1e-3)
    B = synth.multivector(A.n_rows, 8, 2, device="cuda")
    X = torch.zeros_like(B)
    bk.block_krylov_solve(ctx, M, B, X, method="gmres", restart=6, rtol=1e-30, max_iters=4, x0_is_zero=True)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
