mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1
timeout 300 python tools/sweep.py --cfg c2 --ks 16,24,32 --ops spmm > gpurun_out/v4_c2b.jsonl 2>&1
