mkdir -p gpurun_out
for d in 0 4 1 5 2 6 3 7; do for c in 1 2; do
  BK_WIN_DEBUG=$d BK_WIN_CTAS=$c timeout 120 python tools/sweep.py --ops spmm --ks 8,16,32 > gpurun_out/dbg_c2_d${d}_c$c.jsonl 2>&1
done; done
for d in 0 4 1 5; do BK_WIN_DEBUG=$d timeout 120 python tools/sweep.py --cfg c3 --ks 8,16,32 > gpurun_out/dbg_c3_d${d}.jsonl 2>&1; done
