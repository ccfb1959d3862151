// nonlin.cu -- SURVEY.md §8(f) NEXT-3: the nonlinear diffusion-reaction operator of
// Algorithm 1 (§2.2; R29) assembled on the device:
//     f(t,u)_a = sum_b h D_ab (u_a - u_b) + h^3 (u_a - u_a^2) - h^3 sin(1 + t) g_a,
//     D_ab = 1 + (u_a^2 + u_b^2)/2  (Neumann: missing neighbours contribute nothing),
// and the Newton matrix J = shift I + scale Df(u) written into an existing CSR with the
// 7-point lattice pattern.  Lattice: x fastest, row = (z ny + y) nx + x.
#include <cuda_runtime.h>

#include "bk_internal.h"

namespace bk {
namespace {

struct Lat {
    int64_t nx, ny, nz;
};

__device__ __forceinline__ void coords(const Lat& L, int64_t a, int64_t& ix, int64_t& iy, int64_t& iz) {
    ix = a % L.nx;
    const int64_t r = a / L.nx;
    iy = r % L.ny;
    iz = r / L.ny;
}

// F[:, i] = f(T_i, Y[:, i]); thread per (row, column) in row-major order (coalesced)
__global__ void dr_f_kernel(Lat L, double h, const double* __restrict__ Y, int64_t ldy, int w,
                            const double* __restrict__ sinT, const double* __restrict__ g, double* __restrict__ F,
                            int64_t ldf) {
    const int64_t N = L.nx * L.ny * L.nz;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * w) return;
    const int64_t a = e / w;
    const int i = (int)(e - a * w);
    int64_t ix, iy, iz;
    coords(L, a, ix, iy, iz);
    const double ua = Y[a * ldy + i];
    const double h3 = h * h * h;
    double acc = h3 * (ua - ua * ua) - h3 * sinT[i] * g[a];
    const int64_t s1 = L.nx, s2 = L.nx * L.ny;
    const int64_t off[6] = {-s2, -s1, -1, 1, s1, s2};
    const bool has[6] = {iz > 0, iy > 0, ix > 0, ix < L.nx - 1, iy < L.ny - 1, iz < L.nz - 1};
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        if (!has[d]) continue;
        const double ub = Y[(a + off[d]) * ldy + i];
        const double D = 1.0 + 0.5 * (ua * ua + ub * ub);
        acc += h * D * (ua - ub);
    }
    F[a * ldf + i] = acc;
}

// val of J = shift I + scale Df(u) for the CSR (rp, col) with the lattice pattern
__global__ void dr_jac_kernel(Lat L, double h, const double* __restrict__ u, int64_t ldu, double shift,
                              double scale, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                              double* __restrict__ val, int* bad) {
    const int64_t N = L.nx * L.ny * L.nz;
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= N) return;
    int64_t ix, iy, iz;
    coords(L, a, ix, iy, iz);
    const double ua = u[a * ldu];
    const int64_t s1 = L.nx, s2 = L.nx * L.ny;
    const int64_t off[6] = {-s2, -s1, -1, 1, s1, s2};
    const bool has[6] = {iz > 0, iy > 0, ix > 0, ix < L.nx - 1, iy < L.ny - 1, iz < L.nz - 1};
    double diag = shift + scale * h * h * h * (1.0 - 2.0 * ua);
    double offv[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        offv[d] = 0.0;
        if (!has[d]) continue;
        const double ub = u[(a + off[d]) * ldu];
        const double D = 1.0 + 0.5 * (ua * ua + ub * ub);
        diag += scale * h * (D + ua * (ua - ub));
        offv[d] = scale * h * (ub * (ua - ub) - D);
    }
    int found = 0;
    for (int p = rp[a]; p < rp[a + 1]; ++p) {
        const int64_t o = (int64_t)col[p] - a;
        double v = 0.0;
        bool hit = false;
        if (o == 0) { v = diag; hit = true; }
#pragma unroll
        for (int d = 0; d < 6; ++d)
            if (has[d] && o == off[d]) { v = offv[d]; hit = true; }
        val[p] = v;
        found += hit ? 1 : 0;
    }
    int need = 1;
#pragma unroll
    for (int d = 0; d < 6; ++d) need += has[d] ? 1 : 0;
    if (found != need) atomicExch(bad, 1);   // pattern does not hold the stencil
}

}  // namespace

void launch_dr_f(int64_t nx, int64_t ny, int64_t nz, double h, const double* Y, int64_t ldy, int w,
                 const double* sinT, const double* g, double* F, int64_t ldf, cudaStream_t st) {
    const int64_t t = nx * ny * nz * w;
    if (t > 0) BK_KERNEL(dr_f_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(Lat{nx, ny, nz}, h, Y, ldy, w, sinT,
                                                                                    g, F, ldf));
}

void launch_dr_jac(int64_t nx, int64_t ny, int64_t nz, double h, const double* u, int64_t ldu, double shift,
                   double scale, const int32_t* rp, const int32_t* col, double* val, int* bad, cudaStream_t st) {
    const int64_t n = nx * ny * nz;
    if (n > 0) BK_KERNEL(dr_jac_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Lat{nx, ny, nz}, h, u, ldu, shift,
                                                                                    scale, rp, col, val, bad));
}

}  // namespace bk
