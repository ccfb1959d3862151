mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1
timeout 600 python tools/config_sweep.py --cfgs c3,c4 > gpurun_out/cfg_c34.jsonl 2>&1
for r in 0 1; do BK_SPMM_ROLL=$r timeout 300 python tools/sweep.py --cfg c2 --ks 16,32 --ops spmm,spmm_C > gpurun_out/sw_c2_roll$r.jsonl 2>&1; done
