#!/bin/bash
# HEAD ncu captures: RED 1 / RED 2 of the SECOND BiCGStab iteration of a bench step (distinct
# operands), and the 3-D gather kernel's coupled path at k = 32 (c4) with its source page
O=gpurun_out; mkdir -p $O
STEP="python bench.py --profile-step --no-sweep --no-e2e --no-cpu-baseline --no-configs --steps 1 --warmup 3"
for red in 1 2; do
    ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:bspmm_win_kernel -s $((6 + red)) -c 1 -o $O/r2_fused_red$red $STEP > $O/r2_fused_red$red.log 2>&1
    ncu -i $O/r2_fused_red$red.ncu-rep --page raw --csv > $O/r2_fused_red$red.raw.csv 2>/dev/null
    rm -f $O/r2_fused_red$red.ncu-rep
done
python tools/one_apply.py --cfg c4 --k 32 --reps 2 --coupled > $O/e23_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bspmm -s 1 -c 1 -o $O/e23_c4_k32_coupled \
    python tools/one_apply.py --cfg c4 --k 32 --reps 2 --coupled > $O/e23_ncu.log 2>&1
ncu -i $O/e23_c4_k32_coupled.ncu-rep --page raw --csv > $O/e23_c4_k32_coupled.raw.csv 2>/dev/null
ncu -i $O/e23_c4_k32_coupled.ncu-rep --page source --csv > $O/e23_c4_k32_coupled.source.csv 2>/dev/null
rm -f $O/e23_c4_k32_coupled.ncu-rep
ls -la $O | grep -E "e23|fused_red"
