#!/bin/bash
# fused-reduction applies: three 128-consumer CTAs per SM (BK_RED_NC=128) vs two 256-consumer CTAs
O=gpurun_out; mkdir -p $O; rm -f $O/e13_class.jsonl
BK_RED_NC=128 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py tests/test_gpu_cg1.py -m gpu -q -x -k "bicgstab or fused or cg" > $O/e13_tests.log 2>&1; tail -2 $O/e13_tests.log
for nc in 256 128; do
for k in 8 12 16; do BK_RED_NC=$nc python tools/class_timing.py --cfg c2 --k $k --method bicgstab --tag nc$nc >> $O/e13_class.jsonl; done
for m in cg cg1; do BK_RED_NC=$nc python tools/class_timing.py --cfg c2s --k 16 --method $m --tag nc$nc >> $O/e13_class.jsonl; done
done
python - <<'PY'
import json
for l in open("gpurun_out/e13_class.jsonl"):
    d = json.loads(l); u = d["us_per_launch"]
    print(d["tag"], d["method"], d["k"], {k: v for k, v in u.items() if k.startswith("fused")})
PY
