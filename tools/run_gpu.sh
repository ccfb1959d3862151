mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --profile-step --steps 1 --warmup 3 --no-sweep --no-e2e --no-configs > gpurun_out/ncu_step.log 2>&1
timeout 300 python tools/alg1_timing.py > gpurun_out/alg1_c3.jsonl 2>&1
