mkdir -p gpurun_out
timeout 600 python tools/alg1_timing.py --rtol 1e-5 --steps 3 --windows 1,3 > gpurun_out/alg1_c3_r5.jsonl 2>&1
timeout 600 python tools/alg1_timing.py --rtol 1e-5 --steps 3 --windows 1,3 --method gmres > gpurun_out/alg1_c3_r5g.jsonl 2>&1
