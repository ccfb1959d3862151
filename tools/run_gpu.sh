# Reproduce the round's GPU evidence on a B200 box (gpurun -- 'bash tools/run_gpu.sh'):
# parity tests, smoke, the bench line, the launch list of one step (profiles/r01_*).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_step.csv python bench.py --profile-step --steps 1 --warmup 3 --no-sweep \
    --no-e2e --no-configs > gpurun_out/ncu_step.log 2>&1
