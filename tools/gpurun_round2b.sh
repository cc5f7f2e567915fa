#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpurun_ab.sh "4 2 3" tools/ab/lib_base.so tools/ab/lib_fma.so
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu_all.log 2>&1
echo "rc=$?" >> gpurun_out/t_gpu_all.log
