#!/bin/bash
# 2-D plain apply at k = 12 / 24: windowed band kernel (default) vs the gather kernel (BK_SPMM_WIN=0;
# k = 12 has the three-lane instantiation there)
O=gpurun_out; mkdir -p $O; rm -f $O/e22_sweep.jsonl
for w in 1 0; do
  echo "== BK_SPMM_WIN=$w" >> $O/e22_sweep.jsonl
  BK_SPMM_WIN=$w python tools/sweep.py --cfg c2 --ks 8,12,16,20,24,32 --ops spmm,spmm_C --reps 5 | grep -v copy >> $O/e22_sweep.jsonl
done
cat $O/e22_sweep.jsonl
