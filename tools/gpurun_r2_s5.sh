#!/bin/bash
# A/B k_small radix-3 twiddle prefetch (config 2); ncu --set full of the config-1 chain.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
timeout 900 python tools/abtime.py --config 2 --rounds 3 ablibs/lib_base.so ablibs/lib_stwpf.so > gpurun_out/s5_ab_c2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pack|k_pass|k_carry" -c 6 -o /tmp/ncu/s5_cfg1 python tools/profile_case.py --config 1 --reps 1 > gpurun_out/s5_ncu1.log 2>&1
ncu -i /tmp/ncu/s5_cfg1.ncu-rep --page raw --csv > gpurun_out/s5_cfg1_raw.csv 2>/dev/null
ncu -i /tmp/ncu/s5_cfg1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/s5_cfg1_source.csv 2>/dev/null
gzip -f gpurun_out/s5_cfg1_source.csv
grep "==" gpurun_out/s5_ab_c2.txt | cut -c1-300
