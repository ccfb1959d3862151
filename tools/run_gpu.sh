mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gmres or update or solve or dirk or alg1 or wide" > gpurun_out/t_sub.log 2>&1
timeout 300 python tools/solve_timing.py --cfg c3 --k 12 --method gmres --iters 6,12 --restart 6 > gpurun_out/gm_t.log 2>&1
timeout 300 python tools/solve_timing.py --cfg c2 --k 16 --method gmres --iters 6,12 --restart 6 > gpurun_out/gm_t2.log 2>&1
timeout 300 python tools/solve_timing.py --cfg c2 --k 16 --method gmres --iters 20,30 --restart 30 > gpurun_out/gm_t3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_gmres.csv python tools/solve_timing.py --cfg c3 --k 12 --method gmres --iters 3,6 --reps 1 --restart 6 > gpurun_out/gm.log 2>&1
