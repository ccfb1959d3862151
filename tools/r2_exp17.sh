#!/bin/bash
# streaming-ring geometry A/B (stages x KB per stage): fused tails, Grams, updates
O=gpurun_out; mkdir -p $O; rm -f $O/e17_class.jsonl
for lib in default lib_ab/libbk_s3x32.so lib_ab/libbk_s2x56.so lib_ab/libbk_s4x24.so; do
  if [ $lib = default ]; then unset BK_LIB_PATH; else export BK_LIB_PATH=$PWD/paper_2504_02117_b200/$lib; fi
  python tools/class_timing.py --cfg c2 --k 16 --method bicgstab --tag $lib >> $O/e17_class.jsonl
  python tools/class_timing.py --cfg c2s --k 16 --method cg --tag $lib >> $O/e17_class.jsonl
  echo "== $lib"; python tools/sweep.py --cfg c2 --ks 8,16,32 --ops gram,update --reps 5 | grep -v copy
done
python - <<'PY'
import json
for l in open("gpurun_out/e17_class.jsonl"):
    d = json.loads(l); u = d["us_per_launch"]
    print(d["tag"], d["method"], {k: v for k, v in u.items() if k in ("fused_tail", "update", "fused_apply", "fused_apply_dots")})
PY
