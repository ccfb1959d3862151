mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -n 3 gpurun_out/t_all.log
timeout 120 python tools/sweep.py --ops gram > gpurun_out/sw_gram.jsonl 2>&1
BK_GRAM_PANEL=0 timeout 120 python tools/sweep.py --ops gram > gpurun_out/sw_gram0.jsonl 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --profile-step --warmup 3 > gpurun_out/ncu_step.log 2>&1
python tools/ncu_launches.py gpurun_out/launches_step.csv 40 > gpurun_out/launches_step.txt
