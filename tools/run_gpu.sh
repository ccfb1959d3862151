mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cheb or gersh or jacobi or solve_matches" > gpurun_out/t_cheb.log 2>&1
