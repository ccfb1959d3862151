#!/bin/bash
# ncu --set full of the lane-exact gather instantiations on c2 (k = 12, 20, 24)
O=gpurun_out; mkdir -p $O
for k in 12 20 24; do
  tag=e29_apply_c2_k$k
  python tools/one_apply.py --cfg c2 --k $k --reps 2 > $O/$tag.plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bspmm -s 1 -c 1 -o $O/$tag \
      python tools/one_apply.py --cfg c2 --k $k --reps 2 > $O/$tag.log 2>&1
  ncu -i $O/$tag.ncu-rep --page raw --csv > $O/$tag.raw.csv 2>/dev/null
  rm -f $O/$tag.ncu-rep
done
ls $O | grep e29
