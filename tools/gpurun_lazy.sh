#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_multi.py -x -q > gpurun_out/t_lazy.log 2>&1; echo rc=$? >> gpurun_out/t_lazy.log
tail -3 gpurun_out/t_lazy.log
timeout 500 python tools/abtime.py --config 3 --rounds 3 tools/ab/lib_epi3p.so tools/ab/lib_lazy.so > gpurun_out/ab_c3d.txt 2>&1
timeout 500 python tools/abtime.py --config 4 --rounds 2 --steps 5 tools/ab/lib_epi3p.so tools/ab/lib_lazy.so > gpurun_out/ab_c4d.txt 2>&1
timeout 300 python tools/abtime.py --config 33 --rounds 2 tools/ab/lib_epi3p.so tools/ab/lib_lazy.so > gpurun_out/ab_c33d.txt 2>&1
grep "==" gpurun_out/ab_c3d.txt gpurun_out/ab_c4d.txt gpurun_out/ab_c33d.txt | cut -c1-330
grep "ok=" gpurun_out/ab_c*d.txt | grep -v "ok=True" | head
