#!/bin/bash
# k = 20 plain apply: five-lane gather instantiation vs the band kernel (BK_WIN_K20=1) on c2, and on c4
O=gpurun_out; mkdir -p $O; rm -f $O/e28_sweep.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "spmm or coupl or apply" > $O/e28_tests.log 2>&1; tail -2 $O/e28_tests.log
for w in 0 1; do
  echo "== BK_WIN_K20=$w" >> $O/e28_sweep.jsonl
  BK_WIN_K20=$w python tools/sweep.py --cfg c2 --ks 20 --ops spmm --reps 7 | grep -v copy >> $O/e28_sweep.jsonl
done
python tools/sweep.py --cfg c4 --ks 20 --ops spmm --reps 5 | grep -v copy >> $O/e28_sweep.jsonl
cat $O/e28_sweep.jsonl
