// Do the FP64 tensor path (mma.sync f64) and the FP64 FMA path share one pipe on B200?  Half the
// warps of every CTA run DMMA, half DFMA, concurrently; if the sum exceeds either peak alone the
// coupled apply can split its k x k product between them.  Also the larger f64 MMA shapes
// (m16n8k4 / m16n8k8 / m16n8k16, PTX sm_90+).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_mixed tools/micro/fp64_mixed.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;

template <int SHAPE>   // 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
__device__ __forceinline__ void mma_step(double (&d)[CH][4], double a, double b) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        if constexpr (SHAPE == 0)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
        else if constexpr (SHAPE == 1)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3]) : "d"(a), "d"(b), "d"(b));
        else if constexpr (SHAPE == 2)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                         : "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b));
        else
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                         "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                         : "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a),
                           "d"(b));
    }
}

// mode: 0 all warps MMA, 1 all warps DFMA, 2 even warps MMA / odd warps DFMA
template <int SHAPE>
__global__ void loop(double* out, int iters, int mode) {
    const int warp = threadIdx.x >> 5;
    const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
    double d[CH][4];
    const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
    if (do_mma) {
        for (int i = 0; i < iters; ++i) mma_step<SHAPE>(d, a, b);
    } else {
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int c = 0; c < CH; ++c) d[c][0] = fma(d[c][0], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 12345.678) out[0] = s;
}

template <int SHAPE>
void run(const char* name, double mma_flop, int nsm, double* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, blocks = 2 * nsm, threads = 512;
    for (int mode = 0; mode < 3; ++mode) {
        if (SHAPE != 0 && mode == 1) continue;
        loop<SHAPE><<<blocks, threads>>>(out, 100, mode);
        cudaEventRecord(e0);
        loop<SHAPE><<<blocks, threads>>>(out, iters, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warps = (double)blocks * threads / 32;
        const double wm = mode == 0 ? warps : (mode == 1 ? 0 : warps / 2), wf = warps - wm;
        const double fl = (wm * mma_flop + wf * 32 * 2.0) * iters * CH;
        printf("{\"shape\": \"%s\", \"mode\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f}\n", name,
               mode == 0 ? "mma" : (mode == 1 ? "dfma" : "half_mma_half_dfma"), fl / (ms * 1e-3) / 1e12, ms);
    }
    cudaError_t e = cudaGetLastError();
    if (e) printf("{\"shape\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(e));
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    run<0>("m8n8k4", 8 * 8 * 4 * 2, nsm, out);
    run<1>("m16n8k4", 16 * 8 * 4 * 2, nsm, out);
    run<2>("m16n8k8", 16 * 8 * 8 * 2, nsm, out);
    run<3>("m16n8k16", 16 * 8 * 16 * 2, nsm, out);
    return 0;
}
