#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi.py -x -q -p no:cacheprovider --timeout=300 > gpurun_out/t_r10.log 2>&1; echo rc=$? >> gpurun_out/t_r10.log; tail -3 gpurun_out/t_r10.log
timeout 600 python tools/abtime.py --config 5 --rounds 1 --steps 2 tools/ab/lib_base10.so tools/ab/lib_r10.so 2>&1 | grep "=="
timeout 400 python tools/abtime.py --config 4 --rounds 1 --steps 5 tools/ab/lib_base10.so tools/ab/lib_r10.so 2>&1 | grep "=="
timeout 300 python tools/abtime.py --config 3 --rounds 2 tools/ab/lib_base10.so tools/ab/lib_r10.so 2>&1 | grep "=="
