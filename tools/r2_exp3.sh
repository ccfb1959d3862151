#!/bin/bash
# full GPU suite + class timings of CG / CG1 / BiCGStab + bench (round 2, after the in-place update fix)
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/e3_tests.log 2>&1; tail -3 $O/e3_tests.log
for m in cg cg1; do python tools/class_timing.py --method $m --cfg c2s --k 16 >> $O/e3_class.jsonl 2>&1; done
python tools/class_timing.py --method bicgstab --cfg c2 --k 16 >> $O/e3_class.jsonl 2>&1
for cfg in "c2s 8" "c2s 16" "c4 16"; do set -- $cfg
  for m in cg cg1; do timeout 300 python tools/solve_timing.py --cfg $1 --k $2 --method $m --iters 10,30 --reps 3 >> $O/e3_timing.jsonl 2>&1; done
done
cat $O/e3_class.jsonl $O/e3_timing.jsonl
timeout 900 python bench.py > $O/e3_bench.json 2> $O/e3_bench.err; tail -c 600 $O/e3_bench.json
