#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_full.py -q -x -k "flat" > $O/e1_flat.log 2>&1; tail -2 $O/e1_flat.log
timeout 900 python -m pytest tests/test_gpu_cg1.py -q -x -k "byte" > $O/e1_bytes.log 2>&1; tail -2 $O/e1_bytes.log
python tools/sweep.py --cfg c2 --ks 1,2,4 --ops gram,update --reps 5 > $O/e1_sweep.log 2>&1; tail -20 $O/e1_sweep.log
for tr in "" 32 48 64 80 96; do
  for m in bicgstab cg1; do
    BK_WIN_TR=$tr python tools/class_timing.py --method $m --k 16 --cfg $([ $m = cg1 ] && echo c2s || echo c2) >> $O/e1_tr.jsonl 2>>$O/e1_tr.err
  done
done
cat $O/e1_tr.jsonl
