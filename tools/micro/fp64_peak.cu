// FP64 peak of the B200 SM paths this library uses: m8n8k4 DMMA (mma.sync f64,
// the tensor-core path of the Gram / update / coupled-apply kernels) and plain FMA (DFMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/micro/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;   // independent accumulator chains per thread

__global__ void dmma_loop(double* out, int iters) {
    double d[CH][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double d[CH];
    const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) d[c] = fma(d[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = nsm * 2, threads = warps * 32 / 2;
        dmma_loop<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        // per warp-level m8n8k4: 8*8*4 MACs = 512 flop
        const double fl = (double)blocks * (threads / 32) * iters * CH * 512.0;
        printf("{\"path\": \"dmma_m8n8k4_f64\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", warps, fl / (ms * 1e-3) / 1e12);
        dfma_loop<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl2 = (double)blocks * threads * iters * CH * 2.0;
        printf("{\"path\": \"dfma\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", warps, fl2 / (ms * 1e-3) / 1e12);
    }
    return 0;
}
