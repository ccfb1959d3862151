mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -n 3 gpurun_out/t_all.log
timeout 600 python tools/wide_timing.py > gpurun_out/wide_timing.jsonl 2>&1; cat gpurun_out/wide_timing.jsonl
timeout 300 python tools/solve_timing.py --cfg c3 --k 12 --method gmres --restart 32 --iters 4,8 >> gpurun_out/gm.jsonl 2>&1; tail -n 1 gpurun_out/gm.jsonl
