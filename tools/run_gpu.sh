mkdir -p gpurun_out
timeout 900 python tools/dirk_timing.py --n 1024 --s 2,4,8 --method cg --sym --precond chebyshev --inner-rtol 1e-2 --outer-tol 1e-8 > gpurun_out/dirk_t5.jsonl 2>&1
timeout 900 python tools/dirk_timing.py --n 1024 --s 2,4,8 --method bicgstab --inner-rtol 1e-2 --outer-tol 1e-8 --tau 0.001 > gpurun_out/dirk_t6.jsonl 2>&1
