#!/bin/bash
# DMMA chain interleaving (coupled applies, k <= 16 updates): parity + sweep + bench
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -m gpu -q -x -k "spmm or update or apply or coupled or fused or solve" > $O/e6_tests.log 2>&1; tail -3 $O/e6_tests.log
python tools/sweep.py --cfg c2 --ks 8,16,32 --ops spmm,spmm_C,update --reps 5 > $O/e6_sweep.log 2>&1
python tools/sweep.py --cfg c4 --ks 8,16,32 --ops spmm,spmm_C --reps 3 >> $O/e6_sweep.log 2>&1
cat $O/e6_sweep.log | grep -v copy
python tools/one_apply.py --cfg c2 --k 32 --coupled --reps 2 > $O/e6_c32.plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bspmm -s 1 -c 1 -o $O/e6_c32 \
    python tools/one_apply.py --cfg c2 --k 32 --coupled --reps 2 > $O/e6_c32.log 2>&1
ncu -i $O/e6_c32.ncu-rep --page raw --csv > $O/e6_c32.raw.csv 2>/dev/null
ncu -i $O/e6_c32.ncu-rep --page source --csv > $O/e6_c32.source.csv 2>/dev/null
rm -f $O/e6_c32.ncu-rep
timeout 900 python bench.py --no-configs > $O/e6_bench.json 2> $O/e6_bench.err; tail -c 200 $O/e6_bench.json
