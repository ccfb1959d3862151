#!/bin/bash
# Coupled apply with the window's structured coupling (all-zero C fragments skipped): parity, sweep,
# and the fused-apply ncu captures at HEAD
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "coupl or windowed_paths or integer_bitwise or random_within" > $O/e20_tests.log 2>&1
for cfg in c2 c4; do
  python tools/sweep.py --cfg $cfg --ks 8,12,16,24,32 --ops spmm,spmm_C,spmm_Cw --reps 5 | grep -v copy >> $O/e20_sweep.jsonl
done
STEP="python bench.py --profile-step --no-sweep --no-e2e --no-cpu-baseline --no-configs --steps 1 --warmup 3"
for red in 1 2; do
    ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:bspmm_win_kernel -s $((4 + red)) -c 1 -o $O/r2_fused_red$red $STEP > $O/r2_fused_red$red.log 2>&1
    ncu -i $O/r2_fused_red$red.ncu-rep --page raw --csv > $O/r2_fused_red$red.raw.csv 2>/dev/null
    ncu -i $O/r2_fused_red$red.ncu-rep --page details --csv > $O/r2_fused_red$red.details.csv 2>/dev/null
    rm -f $O/r2_fused_red$red.ncu-rep
done
tail -3 $O/e20_tests.log; cat $O/e20_sweep.jsonl
