#!/bin/bash
# Re-check of the twiddle-row L2 prefetch choices after the TMA tiles (config 4).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/abtime.py --config 4 --rounds 3 --steps 5 ablibs/lib_base.so ablibs/lib_noinvpf.so ablibs/lib_fwdpf.so > gpurun_out/s35_ab_c4.txt 2>&1
grep "==" gpurun_out/s35_ab_c4.txt | cut -c1-300
