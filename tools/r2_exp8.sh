#!/bin/bash
# c3 block GMRES(64), k = 12: where one restart cycle's time goes (slope + ncu launch list)
O=gpurun_out; mkdir -p $O
true
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
   --log-file $O/e8_launches.csv python tools/solve_timing.py --cfg c3 --k 12 --method gmres --restart 64 --iters 48 --reps 1 > $O/e8_ncu.log 2>&1
python tools/ncu_launches.py $O/e8_launches.csv | head -40
