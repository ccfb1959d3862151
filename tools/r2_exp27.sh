#!/bin/bash
# k = 24 plain apply: six-lane gather instantiation vs the band kernel (BK_WIN_K24=1) on c2, and on c4 / c3
O=gpurun_out; mkdir -p $O; rm -f $O/e27_sweep.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "spmm or coupl or apply" > $O/e27_tests.log 2>&1; tail -2 $O/e27_tests.log
for w in 0 1; do
  echo "== BK_WIN_K24=$w" >> $O/e27_sweep.jsonl
  BK_WIN_K24=$w python tools/sweep.py --cfg c2 --ks 24 --ops spmm --reps 7 | grep -v copy >> $O/e27_sweep.jsonl
done
python tools/sweep.py --cfg c4 --ks 24 --ops spmm --reps 5 | grep -v copy >> $O/e27_sweep.jsonl
python tools/sweep.py --cfg c3 --ks 24 --ops spmm --reps 5 | grep -v copy >> $O/e27_sweep.jsonl
cat $O/e27_sweep.jsonl
