#!/bin/bash
# wide update: H fragments first, column split beyond a 32-row tile; GMRES parity + c3 GMRES(64) cycle time
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -m gpu -q -x -k "update or gmres or gram" > $O/e9_tests.log 2>&1; tail -3 $O/e9_tests.log
python tools/solve_timing.py --cfg c3 --k 12 --method gmres --restart 64 --iters 16,32,64 --reps 2 > $O/e9_slope.json 2>&1; cat $O/e9_slope.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/e9_launches.csv python tools/solve_timing.py --cfg c3 --k 12 --method gmres --restart 64 --iters 48 --reps 1 > $O/e9_ncu.log 2>&1
python tools/ncu_launches.py $O/e9_launches.csv | grep "bk::" | head -20
