#!/bin/bash
# L2 prefetch (leading band segment, streamed rows, CSR of the next tile): BK_RED_PF for the
# fused-reduction applies, BK_WIN_PF for the plain windowed apply
O=gpurun_out; mkdir -p $O; rm -f $O/e19_class.jsonl
for pf in 0 1 2; do
  for k in 16 12 8; do
    BK_RED_PF=$pf python tools/class_timing.py --cfg c2 --k $k --method bicgstab --tag pf$pf >> $O/e19_class.jsonl
  done
  BK_RED_PF=$pf python tools/class_timing.py --cfg c2s --k 16 --method cg --tag pf$pf >> $O/e19_class.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/e19_class.jsonl"):
    d = json.loads(l); u = d["us_per_launch"]
    print(d["tag"], d["method"], d["k"], {k: v for k, v in u.items() if k.startswith("fused") or k == "update"})
PY
for pf in 0 1 2; do echo "== BK_WIN_PF=$pf"; BK_WIN_PF=$pf python tools/sweep.py --cfg c2 --ks 4,8,16,32 --ops spmm --reps 5 | grep -v copy; done
