#!/bin/bash
# solver tests after the B-in-place setup + bench + c3 GMRES(64) repeat + sanitizers
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py tests/test_gpu_cg1.py tests/test_gpu_multirank.py -m gpu -q -x -k "solve or solver or cg1 or fused or bicgstab or dirk or alg1 or cheb or graph or byte" > $O/e4_tests.log 2>&1; tail -3 $O/e4_tests.log
timeout 900 python bench.py --no-configs > $O/e4_bench.json 2> $O/e4_bench.err; tail -c 300 $O/e4_bench.json
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_case.py > $O/e4_racecheck.log 2>&1; tail -5 $O/e4_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_case.py > $O/e4_synccheck.log 2>&1; tail -5 $O/e4_synccheck.log
