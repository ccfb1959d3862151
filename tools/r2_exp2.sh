#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/class_timing.py --method cg --cfg c2s --k 16 > $O/e2_cg_class.json 2>&1; cat $O/e2_cg_class.json
for m in cg cg1; do
  ncu --set full --clock-control none --import-source on -k regex:bspmm_win --launch-skip 2 -c 1 -o $O/e2_$m \
      python tools/class_timing.py --method $m --cfg c2s --k 16 --iters 3 > $O/e2_$m.log 2>&1
  ncu -i $O/e2_$m.ncu-rep --page raw --csv > $O/e2_$m.raw.csv 2>/dev/null
  ncu -i $O/e2_$m.ncu-rep --page source --csv --print-source cuda > $O/e2_$m.cuda.csv 2>/dev/null
  rm -f $O/e2_$m.ncu-rep
done
SW="python tools/sweep.py --cfg c2 --ks 1,2,4 --ops gram,update --reps 2"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control all \
    --clock-control none --csv --log-file $O/e2_small.csv -k regex:"flat|vec" $SW > $O/e2_small.log 2>&1
