#!/bin/bash
# fused-reduction applies with tiles a multiple of one pass's rows; plain apply tile A/B
O=gpurun_out; mkdir -p $O; rm -f $O/e12_class.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py tests/test_gpu_cg1.py -m gpu -q -x -k "bicgstab or fused or cg" > $O/e12_tests.log 2>&1; tail -2 $O/e12_tests.log
for k in 8 12 16; do python tools/class_timing.py --cfg c2 --k $k --method bicgstab --tag rpp >> $O/e12_class.jsonl; done
for m in cg cg1; do for k in 8 16; do python tools/class_timing.py --cfg c2s --k $k --method $m --tag rpp >> $O/e12_class.jsonl; done; done
python - <<'PY'
import json
for l in open("gpurun_out/e12_class.jsonl"):
    d = json.loads(l); u = d["us_per_launch"]
    print(d["method"], d["k"], {k: v for k, v in u.items() if k.startswith("fused")})
PY
python tools/sweep.py --cfg c2 --ks 8,16 --ops spmm --reps 7
BK_WIN_TR=64 python tools/sweep.py --cfg c2 --ks 16 --ops spmm --reps 7
BK_WIN_TR=128 python tools/sweep.py --cfg c2 --ks 8 --ops spmm --reps 7
