#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi.py -x -q > gpurun_out/t_r3f.log 2>&1; echo rc=$? >> gpurun_out/t_r3f.log
tail -3 gpurun_out/t_r3f.log
timeout 500 python tools/abtime.py --config 4 --rounds 2 --steps 5 tools/ab/lib_f2.so tools/ab/lib_r3f.so > gpurun_out/ab_c4h.txt 2>&1
DECMUL_R3_FULL=0 timeout 500 python tools/abtime.py --config 4 --rounds 1 --steps 5 tools/ab/lib_r3f.so > gpurun_out/ab_c4h0.txt 2>&1
grep "==" gpurun_out/ab_c4h.txt gpurun_out/ab_c4h0.txt | cut -c1-330
grep "ok=" gpurun_out/ab_c*h*.txt | grep -v "ok=True" | head
