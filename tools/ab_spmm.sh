# A/B of bspmm variants (env BK_SPMM_KERNEL / BK_SPMM_VEC) with tools/sweep.py; results in gpurun_out/ab.jsonl
set -o pipefail
for kern in ${KERNS:-pipe pipe4x2 pipe4x3t128 pipe8x3t128n128 pipe3x2n384}; do for v in ${VECS:-4}; do
  BK_SPMM_KERNEL=$kern BK_SPMM_VEC=$v timeout 120 python tools/sweep.py --ops spmm >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
  BK_SPMM_KERNEL=$kern BK_SPMM_VEC=$v timeout 120 python tools/sweep.py --cfg c3 --ks 1,4,8,12,16,32 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done; done
