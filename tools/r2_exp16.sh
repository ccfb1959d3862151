#!/bin/bash
# register (row-per-lane) k x k solvers: whole GPU suite + solver iteration timings + k x k kernel durations
O=gpurun_out; mkdir -p $O; rm -f $O/e16_class.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > $O/e16_tests.log 2>&1; tail -3 $O/e16_tests.log
for k in 8 16; do python tools/class_timing.py --cfg c2 --k $k --method bicgstab --tag reglu >> $O/e16_class.jsonl; done
for m in cg cg1; do python tools/class_timing.py --cfg c2s --k 16 --method $m --tag reglu >> $O/e16_class.jsonl; done
cat $O/e16_class.jsonl
python tools/solve_timing.py --cfg c2 --k 16 --method bicgstab --iters 5,10,20
python tools/solve_timing.py --cfg c2s --k 16 --method cg --iters 5,10,20
python tools/solve_timing.py --cfg c2s --k 16 --method cg1 --iters 5,10,20
bash tools/r2_exp15.sh
