#!/bin/bash
# GPU check of the single-reduction block CG: parity tests, per-iteration timing vs block CG,
# ncu of the fused BiCGStab applies (RED 1 / RED 2: 6th / 7th windowed launch of a bench step)
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cg1.py -q -x > $O/cg1_tests.log 2>&1; tail -3 $O/cg1_tests.log
for cfg in "c2s 8" "c2s 16" "c4 16"; do
    set -- $cfg
    for m in cg cg1; do
        timeout 300 python tools/solve_timing.py --cfg $1 --k $2 --method $m --iters 10,30 --reps 3 >> $O/cg1_timing.jsonl 2>> $O/cg1_timing.err
    done
done
cat $O/cg1_timing.jsonl
STEP="python bench.py --profile-step --no-sweep --no-e2e --no-cpu-baseline --no-configs --steps 1 --warmup 3"
for sk in 5 6; do
    ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:bspmm_win \
        --launch-skip $sk -c 1 -o $O/r2_fused_skip$sk $STEP > $O/r2_fused_skip$sk.log 2>&1
    ncu -i $O/r2_fused_skip$sk.ncu-rep --page raw --csv > $O/r2_fused_skip$sk.raw.csv 2>/dev/null
    ncu -i $O/r2_fused_skip$sk.ncu-rep --page source --csv > $O/r2_fused_skip$sk.source.csv 2>/dev/null
    rm -f $O/r2_fused_skip$sk.ncu-rep
done
