#!/bin/bash
# fused-apply fragment-load change: parity of every RED path + class timings + ncu lines
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_cg1.py tests/test_gpu_parity.py -m gpu -q -x -k "fused or cg1 or solve or bicgstab" > $O/e5_tests.log 2>&1; tail -3 $O/e5_tests.log
python tools/class_timing.py --method bicgstab --cfg c2 --k 16 > $O/e5_class.jsonl 2>&1
python tools/class_timing.py --method bicgstab --cfg c2 --k 8 >> $O/e5_class.jsonl 2>&1
python tools/class_timing.py --method cg --cfg c2s --k 16 >> $O/e5_class.jsonl 2>&1
python tools/class_timing.py --method cg1 --cfg c2s --k 16 >> $O/e5_class.jsonl 2>&1
BK_RED_CTAS=1 python tools/class_timing.py --method bicgstab --cfg c2 --k 16 --tag ctas1 >> $O/e5_class.jsonl 2>&1
BK_RED_CTAS=1 python tools/class_timing.py --method cg1 --cfg c2s --k 16 --tag ctas1 >> $O/e5_class.jsonl 2>&1
cat $O/e5_class.jsonl
for spec in "bicgstab c2 2 red1" "bicgstab c2 3 red2" "cg1 c2s 2 red4"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:bspmm_win --launch-skip $3 -c 1 -o $O/e5_$4 \
      python tools/class_timing.py --method $1 --cfg $2 --k 16 --iters 3 > $O/e5_$4.log 2>&1
  ncu -i $O/e5_$4.ncu-rep --page raw --csv > $O/e5_$4.raw.csv 2>/dev/null
  ncu -i $O/e5_$4.ncu-rep --page source --csv > $O/e5_$4.source.csv 2>/dev/null
  rm -f $O/e5_$4.ncu-rep
done
