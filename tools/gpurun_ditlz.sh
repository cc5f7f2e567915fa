#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi.py tests/test_gpu_cpp.py -x -q > gpurun_out/t_ditlz.log 2>&1; echo rc=$? >> gpurun_out/t_ditlz.log
tail -3 gpurun_out/t_ditlz.log
timeout 500 python tools/abtime.py --config 3 --rounds 3 tools/ab/lib_lazy.so tools/ab/lib_ditlz.so > gpurun_out/ab_c3e.txt 2>&1
timeout 500 python tools/abtime.py --config 4 --rounds 2 --steps 5 tools/ab/lib_lazy.so tools/ab/lib_ditlz.so > gpurun_out/ab_c4e.txt 2>&1
timeout 300 python tools/abtime.py --config 2 --rounds 3 tools/ab/lib_lazy.so tools/ab/lib_ditlz.so > gpurun_out/ab_c2e.txt 2>&1
grep "==" gpurun_out/ab_c3e.txt gpurun_out/ab_c4e.txt gpurun_out/ab_c2e.txt | cut -c1-330
grep "ok=" gpurun_out/ab_c*e.txt | grep -v "ok=True" | grep -v "ok=None" | head
