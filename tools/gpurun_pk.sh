#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not config5" > gpurun_out/t_pk.log 2>&1; echo rc=$? >> gpurun_out/t_pk.log
tail -3 gpurun_out/t_pk.log
timeout 500 python tools/abtime.py --config 4 --rounds 2 --steps 5 tools/ab/lib_ditlz.so tools/ab/lib_pk.so > gpurun_out/ab_c4f.txt 2>&1
timeout 500 python tools/abtime.py --config 5 --rounds 1 --steps 2 tools/ab/lib_ditlz.so tools/ab/lib_pk.so > gpurun_out/ab_c5f.txt 2>&1
grep "==" gpurun_out/ab_c4f.txt gpurun_out/ab_c5f.txt | cut -c1-330
grep "ok=" gpurun_out/ab_c*f.txt | grep -v "ok=True" | head
