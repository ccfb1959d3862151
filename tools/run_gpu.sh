mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1
timeout 300 python tools/solve_timing.py --cfg c2 --k 16 --method bicgstab > gpurun_out/st_bcg.log 2>&1
