#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi.py -x -q -p no:cacheprovider --timeout=200 > gpurun_out/t_merge.log 2>&1; echo rc=$? >> gpurun_out/t_merge.log; tail -3 gpurun_out/t_merge.log
DECMUL_R3_MERGE=0 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=200 -k "radix3 or fused_pack or sizes_across or lean or large_prime or factorised" 2>&1 | tail -1
timeout 400 python tools/abtime.py --config 4 --rounds 2 --steps 5 tools/ab/lib_pm.so tools/ab/lib_merge2.so 2>&1 | grep "=="
timeout 400 python tools/abtime.py --config 5 --rounds 1 --steps 2 tools/ab/lib_pm.so tools/ab/lib_merge2.so 2>&1 | grep "=="
grep "ok=" gpurun_out/*.txt 2>/dev/null | tail -0
