#!/bin/bash
# device time of the k x k steps as separate kernels (BK_EPI=0): LU solve / re-solve / omega / Cholesky
O=gpurun_out; mkdir -p $O
for m in bicgstab cg; do
cfg=c2; [ $m = cg ] && cfg=c2s
BK_EPI=0 python tools/solve_timing.py --cfg $cfg --k 16 --method $m --iters 5 --reps 1 > /dev/null 2>&1 && \
BK_EPI=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e15_$m.csv \
  python tools/solve_timing.py --cfg $cfg --k 16 --method $m --iters 5 --reps 1 > $O/e15_$m.log 2>&1
python tools/ncu_launches.py $O/e15_$m.csv | grep "bk::" | head -14
done
