#!/bin/bash
# c1 block GMRES(100), k = 4: wide basis kernels vs the generic ones (BK_WIDE=0) at n = 1024
O=gpurun_out; mkdir -p $O
python tools/solve_timing.py --cfg c1 --k 4 --method gmres --restart 100 --iters 10,40 --reps 3
BK_WIDE=0 python tools/solve_timing.py --cfg c1 --k 4 --method gmres --restart 100 --iters 10,40 --reps 3
BK_WIDE=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e11_c1_launches.csv \
  python tools/solve_timing.py --cfg c1 --k 4 --method gmres --restart 100 --iters 20 --reps 1 > $O/e11_c1.log 2>&1
python tools/ncu_launches.py $O/e11_c1_launches.csv | grep "bk::" | head -16
