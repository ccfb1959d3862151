#!/bin/bash
# fused BiCGStab applies (RED 1 / 2): tile rows vs ring stages (BK_WIN_TR) on c2, k = 16 / 8
O=gpurun_out; mkdir -p $O; rm -f $O/e10_class.jsonl
for tr in 0 32 48 64 96; do
  BK_WIN_TR=$tr python tools/class_timing.py --cfg c2 --k 16 --method bicgstab --tag tr$tr >> $O/e10_class.jsonl 2>>$O/e10_err.log
  BK_WIN_TR=$tr python tools/class_timing.py --cfg c2 --k 8 --method bicgstab --tag tr$tr >> $O/e10_class.jsonl 2>>$O/e10_err.log
done
python - <<'PY'
import json
for l in open("gpurun_out/e10_class.jsonl"):
    d = json.loads(l); u = d["us_per_launch"]
    print(d["tag"], d["k"], "RED1", u.get("fused_apply"), "RED2", u.get("fused_apply_dots"), "tail", u.get("fused_tail"))
PY
# c1 block GMRES(100), k = 4: per-kernel device time (launch-bound solve)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e10_c1_launches.csv \
  python tools/solve_timing.py --cfg c1 --k 4 --method gmres --restart 100 --iters 20 --reps 1 > $O/e10_c1.log 2>&1
python tools/ncu_launches.py $O/e10_c1_launches.csv | head -25
python tools/solve_timing.py --cfg c1 --k 4 --method gmres --restart 100 --iters 10,40 --reps 3
