#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi.py -x -q > gpurun_out/t_f2.log 2>&1; echo rc=$? >> gpurun_out/t_f2.log
tail -3 gpurun_out/t_f2.log
timeout 500 python tools/abtime.py --config 4 --rounds 2 --steps 5 tools/ab/lib_pk.so tools/ab/lib_f2.so > gpurun_out/ab_c4g.txt 2>&1
timeout 500 python tools/abtime.py --config 3 --rounds 2 tools/ab/lib_pk.so tools/ab/lib_f2.so > gpurun_out/ab_c3g.txt 2>&1
timeout 300 python tools/abtime.py --config 1 --rounds 2 --steps 50 tools/ab/lib_pk.so tools/ab/lib_f2.so > gpurun_out/ab_c1g.txt 2>&1
grep "==" gpurun_out/ab_c4g.txt gpurun_out/ab_c3g.txt gpurun_out/ab_c1g.txt | cut -c1-330
grep "ok=" gpurun_out/ab_c*g.txt | grep -v "ok=True" | head
