#!/bin/bash
# L2 bulk prefetch of the fused-reduction applies' streamed rows / X segments, pf tiles ahead (BK_RED_PF)
O=gpurun_out; mkdir -p $O; rm -f $O/e18_class.jsonl
for pf in 0 1 2 3 4 6; do
  for m in bicgstab; do
    BK_RED_PF=$pf python tools/class_timing.py --cfg c2 --k 16 --method $m --tag pf$pf >> $O/e18_class.jsonl
    BK_RED_PF=$pf python tools/class_timing.py --cfg c2 --k 8 --method $m --tag pf$pf >> $O/e18_class.jsonl
  done
done
BK_RED_PF=2 python tools/class_timing.py --cfg c2s --k 16 --method cg --tag pf2 >> $O/e18_class.jsonl
BK_RED_PF=0 python tools/class_timing.py --cfg c2s --k 16 --method cg --tag pf0 >> $O/e18_class.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/e18_class.jsonl"):
    d = json.loads(l); u = d["us_per_launch"]
    print(d["tag"], d["method"], d["k"], {k: v for k, v in u.items() if k.startswith("fused") or k == "update"})
PY
