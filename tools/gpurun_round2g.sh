#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "sizes_across or lean or large_prime or forced" > gpurun_out/t_g.log 2>&1
echo "rc=$?" >> gpurun_out/t_g.log
bash tools/gpurun_ab.sh "4" tools/ab/lib_nodb.so tools/ab/lib_pk2.so
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pack_radix3|k_pass_fwd|k_pass_inv|k_pass_fused|k_carry_split_r3|k_carry_emit" -c 9 -o gpurun_out/r02_mid python tools/profile_case.py --config 4 --digits 47000000 --reps 1 > gpurun_out/ncu_mid.log 2>&1
ls -la gpurun_out | head -5
