#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not config5" > gpurun_out/t_fuse.log 2>&1
echo "rc=$?" >> gpurun_out/t_fuse.log
bash tools/gpurun_ab.sh "4 3" tools/ab/lib_base.so tools/ab/lib_fuse.so tools/ab/lib_inv3.so
