#!/bin/bash
# TMA L2 prefetch of the inverse row passes' shared twiddle tables (configs 3, 4, 5).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python tools/abtime.py --config 3 --rounds 3 ablibs/lib_base.so ablibs/lib_invpf.so > gpurun_out/s39_ab_c3.txt 2>&1
timeout 900 python tools/abtime.py --config 4 --rounds 3 --steps 5 ablibs/lib_base.so ablibs/lib_invpf.so > gpurun_out/s39_ab_c4.txt 2>&1
timeout 900 python tools/abtime.py --config 5 --rounds 2 --steps 2 ablibs/lib_base.so ablibs/lib_invpf.so > gpurun_out/s39_ab_c5.txt 2>&1
grep "==" gpurun_out/s39_ab_c*.txt | cut -c1-300
