// reduce.cuh -- the deterministic grid reduction of the streaming passes (stream.cu) and of the
// fused apply + Gram passes (spmm.cu): per-warp partials in shared memory -> fixed-order CTA
// partial -> two-level fixed-order ticket tree (the last CTA of each group of 16, then the last
// group) -> outputs.  One launch, bitwise reproducible, no atomics on data.  Internal header.
#pragma once

#include "bk_internal.h"

namespace bk {

// Output description of a reduction (the fields grid_reduce reads; GramStream carries the same).
struct RedOut {
    double* part = nullptr;   // [gridDim.x + groups][NOUT] partials (stream_part_doubles)
    int* ticket = nullptr;    // zeroed device counters (1 + groups)
    double* G = nullptr;      // mode 0: ka x kb; coldot: d[k]
    double* G2 = nullptr;     // coldot second output
    int mode = 2;             // 0 gram, 2 multi-operand (k x k blocks + column dots)
    int ka = 0, kb = 0, kw = 0;
    double* blk[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
    double* dots[2] = {nullptr, nullptr};
};

// fixed-order cross-warp combine -> CTA partial -> last CTA sums partials in order
// returns true in the CTA that wrote the final outputs (after a CTA barrier)
template <int NC, int NOUT, class GS>
__device__ __forceinline__ bool grid_reduce(const GS& Gs, double* s_red, int nout_real, int kb_real, int ld_out,
                                            bool coldot) {
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __syncwarp();
    // (caller has written s_red[warp * NOUT + o])
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    double* out = Gs.part + (int64_t)blockIdx.x * NOUT;
    for (int o = tid; o < NOUT; o += NC) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NC / 32; ++w) s += s_red[w * NOUT + o];
        out[o] = s;
    }
    // two-level fixed-order tree: the last CTA of each group of RG CTAs sums its
    // group's partials, the last group reducer sums the group results.  Every
    // sum has <= RG terms loaded in one batch (one L2 round trip per level).
    constexpr int RG = 16;
    const int nblk = gridDim.x;
    const int ngrp = (nblk + RG - 1) / RG;
    const int g = blockIdx.x / RG;
    const int gsz = (nblk - g * RG) < RG ? (nblk - g * RG) : RG;
    double* P2 = Gs.part + (int64_t)nblk * NOUT;
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    if (tid == 0) s_last = (atomicAdd(Gs.ticket + 1 + g, 1) == gsz - 1);
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    if (!s_last) return false;
    __threadfence();
    for (int o = tid; o < NOUT; o += NC) {
        double v[RG];
#pragma unroll
        for (int b = 0; b < RG; ++b) v[b] = b < gsz ? __ldcg(Gs.part + (int64_t)(g * RG + b) * NOUT + o) : 0.0;
        double s = v[0];
#pragma unroll
        for (int b = 1; b < RG; ++b) s += v[b];
        P2[(int64_t)g * NOUT + o] = s;
    }
    if (tid == 0) Gs.ticket[1 + g] = 0;
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    if (tid == 0) s_last = (atomicAdd(Gs.ticket, 1) == ngrp - 1);
    asm volatile("bar.sync 1, %0;" ::"r"(NC));
    if (!s_last) return false;
    __threadfence();
    for (int o = tid; o < nout_real; o += NC) {
        int idx, dst;
        double* G;
        if (coldot) {
            const int which = o / kb_real, c = o % kb_real;
            idx = which * 32 + c;
            dst = c;
            G = which ? Gs.G2 : Gs.G;
        } else if (Gs.mode == 2) {
            if (o < Gs.ka * Gs.kb) {
                const int a = o / kb_real, b = o % kb_real;
                idx = a * ld_out + b;
                dst = (a % Gs.kw) * Gs.kw + (b % Gs.kw);
                G = Gs.blk[a / Gs.kw][b / Gs.kw];
            } else {   // column dots after the Gram block (NOUT - 64 + q * 32 + c)
                const int o2 = o - Gs.ka * Gs.kb, q = o2 / Gs.kw, c = o2 % Gs.kw;
                idx = NOUT - 64 + q * 32 + c;
                dst = c;
                G = Gs.dots[q];
            }
            if (!G) continue;
        } else {
            const int a = o / kb_real, b = o % kb_real;
            idx = a * ld_out + b;
            dst = a * kb_real + b;
            G = Gs.G;
        }
        constexpr int MAXG = 32;   // up to 512 CTAs
        double v[MAXG];
#pragma unroll
        for (int q = 0; q < MAXG; ++q) v[q] = q < ngrp ? __ldcg(P2 + (int64_t)q * NOUT + idx) : 0.0;
        double s = v[0];
#pragma unroll
        for (int q = 1; q < MAXG; ++q) s += v[q];
        G[dst] = s;
    }
    if (tid == 0) *Gs.ticket = 0;
    asm volatile("bar.sync 1, %0;" ::"r"(NC));   // final outputs visible to the CTA (epilogue)
    (void)lane;
    (void)warp;
    return true;
}


}  // namespace bk
