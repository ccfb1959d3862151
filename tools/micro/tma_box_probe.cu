// Which 2-D fp64 TMA boxes (bw columns x T rows, ld = 780 doubles) does cuTensorMapEncodeTiled accept?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
    double* p; cudaMalloc(&p, (size_t)780 * 4096 * 8);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
    for (int T : {8, 16, 20, 32, 64}) {
        printf("T=%3d fails at bw:", T);
        for (int bw = 8; bw <= 256; bw += 2) {
            CUtensorMap m;
            cuuint64_t dims[2] = {(cuuint64_t)bw, 4096}; cuuint64_t strides[1] = {780 * 8};
            cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)T}; cuuint32_t es[2] = {1, 1};
            CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) printf(" %d", bw);
        }
        printf("\n");
    }
    return 0;
}
