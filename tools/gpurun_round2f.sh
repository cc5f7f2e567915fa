#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q > gpurun_out/t_f.log 2>&1
echo "rc=$?" >> gpurun_out/t_f.log
bash tools/gpurun_ab.sh "4" tools/ab/lib_inv3.so tools/ab/lib_now2.so tools/ab/lib_nodb.so
bash tools/gpurun_ab.sh "2" tools/ab/lib_now2.so tools/ab/lib_smallpf.so
timeout 600 python tools/abtime.py --config 5 --rounds 1 --steps 2 tools/ab/lib_inv3.so tools/ab/lib_now2.so > gpurun_out/ab_cfg5.txt 2>&1
ls -la gpurun_out
