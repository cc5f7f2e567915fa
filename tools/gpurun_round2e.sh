#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/abtime.py --config 4 --rounds 1 --steps 3 tools/ab/lib_now.so > gpurun_out/ab_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all_e.log 2>&1
echo "rc=$?" >> gpurun_out/t_all_e.log
bash tools/gpurun_ab.sh "4" tools/ab/lib_inv3.so tools/ab/lib_nop32.so tools/ab/lib_now.so
ls -la gpurun_out
