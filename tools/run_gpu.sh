mkdir -p gpurun_out
for rep in 1 2; do for s in 0 1; do BK_SLAB=$s timeout 300 python tools/sweep.py --cfg c5 --ks 16 --ops spmm > gpurun_out/c5ab_${s}_$rep.jsonl 2>&1; done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi.txt
