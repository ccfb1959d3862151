#!/bin/bash
# Round-2 ncu evidence at HEAD (run on the GPU box from the repo root; one ncu family per call).
#   1. launch list of ONE bench step (cold-cache, serialised: kernel shares)
#   2. ncu --set full of the dominant kernel of the step (fused BiCGStab tail)
#   3. ncu --set full of the apply kernels at the BASELINE points (c2 k=16 / k=32, c3 k=12, c5 k=16 / k=32)
#   4. device durations of the narrow (k <= 4) Gram / update kernels on c2 (cold cache)
# Each profiled command first exits 0 without ncu (the recipe in B200_PROFILING.md).
set -u
O=gpurun_out
# reports are exported to CSV and deleted (gpurun brings back <= 64 MiB)
export_rep() {
    ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
    ncu -i $O/$1.ncu-rep --page details --csv > $O/$1.details.csv 2>/dev/null
    rm -f $O/$1.ncu-rep
}
STEP="python bench.py --profile-step --no-sweep --no-e2e --no-cpu-baseline --no-configs --steps 1 --warmup 3"
$STEP > $O/r2_step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/r2_launches.csv $STEP > $O/r2_launches.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:bcg_tail -c 1 \
    -o $O/r2_bcg_tail $STEP > $O/r2_bcg_tail.log 2>&1
export_rep r2_bcg_tail
# the fused apply + reduction kernels of the BiCGStab iteration (RED 1: Rt^T[V R]; RED 2: Rt^T T, dots)
# (the step's windowed-apply launches in order: plain k = 1, 2, 4, 8, 16, then RED 1, RED 2, RED 1, ...;
# the SECOND iteration's launches are taken: in the first one P, R and Rt all alias B)
for red in 1 2; do
    ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:bspmm_win_kernel -s $((6 + red)) -c 1 -o $O/r2_fused_red$red $STEP \
        > $O/r2_fused_red$red.log 2>&1
    export_rep r2_fused_red$red
done
for cfg in "c2 16" "c2 32" "c3 12" "c5 16" "c5 32"; do
    set -- $cfg
    tag=r2_apply_$1_k$2
    python tools/one_apply.py --cfg $1 --k $2 --reps 2 > $O/$tag.plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:bspmm -s 1 -c 1 -o $O/$tag \
        python tools/one_apply.py --cfg $1 --k $2 --reps 2 > $O/$tag.log 2>&1
    export_rep $tag
done
SW="python tools/sweep.py --cfg c2 --ks 1,2,3,4 --ops gram,update --reps 2"
$SW > $O/r2_small_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control all \
    --clock-control none --csv --log-file $O/r2_small.csv -k regex:flat $SW > $O/r2_small.log 2>&1
echo done
