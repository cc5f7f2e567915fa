#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not config5" > gpurun_out/t_cur.log 2>&1
echo "rc=$?" >> gpurun_out/t_cur.log
bash tools/gpurun_ab.sh "4 1" tools/ab/lib_inv3.so tools/ab/lib_cur.so
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pack_radix3|k_pass_fused|k_pass_inv|k_carry_split_r3|k_carry_emit" -c 7 -o gpurun_out/r02_cfg4_a python tools/profile_case.py --config 4 --reps 1 > gpurun_out/ncu_a.log 2>&1
ls -la gpurun_out
