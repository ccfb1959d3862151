#!/bin/bash
# RED 1 / 2 fused applies: Rt (, R) fragments loaded by the consumers one pass ahead (EDIR) vs staged
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -m gpu -q -x -k "bicgstab or fused" > $O/e7_tests.log 2>&1; tail -3 $O/e7_tests.log
for e in 0 1; do for k in 8 12 16; do
  BK_RED_EDIR=$e python tools/class_timing.py --cfg c2 --k $k --method bicgstab --tag edir$e >> $O/e7_class.jsonl 2>>$O/e7_err.log
done; done
cat $O/e7_class.jsonl
BK_RED_EDIR=1 timeout 900 python bench.py --no-configs --no-sweep > $O/e7_bench.json 2> $O/e7_bench.err; tail -c 300 $O/e7_bench.json
