#!/bin/bash
# coupled apply k > 16: DMMA blocks pair two one-pass tiles
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -m gpu -q -x -k "spmm or coupled or apply" > $O/e14_tests.log 2>&1; tail -2 $O/e14_tests.log
python tools/sweep.py --cfg c2 --ks 8,16,24,32 --ops spmm_C --reps 7 | grep -v copy
python tools/sweep.py --cfg c4 --ks 32 --ops spmm_C --reps 3 | grep -v copy
python tools/one_apply.py --cfg c2 --k 32 --coupled --reps 2 > /dev/null 2>&1 && bash tools/ncu_cap.sh r2_coupled_c2_k32_pair bspmm python tools/one_apply.py --cfg c2 --k 32 --coupled --reps 2
python tools/ncu_raw_summary.py $O/r2_coupled_c2_k32_pair.raw.csv | head -6
