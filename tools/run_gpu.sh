mkdir -p gpurun_out
for mb in 3 2; do for w in 0 1; do
  BK_SPMM_WIN=0 BK_PIPE_WALK=$w BK_PIPE_MINB=$mb timeout 300 python tools/sweep.py --cfg c2 --ks 4,8,16,32 --ops spmm > gpurun_out/walk_c2_m${mb}_w${w}.jsonl 2>&1
done; done
for mb in 3 2; do BK_PIPE_WALK=1 BK_PIPE_MINB=$mb timeout 300 python tools/sweep.py --cfg c4 --ks 8,16,32 --ops spmm > gpurun_out/walk_c4_m${mb}.jsonl 2>&1; done
