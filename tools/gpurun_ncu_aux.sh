#!/bin/bash
# ncu --set full of config 4's auxiliary kernels (pack_radix3, column pass, carry chain); CSV export on the box
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_aux.log 2>&1; echo rc=$? >> gpurun_out/t_aux.log; tail -2 gpurun_out/t_aux.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pack_radix3|k_pass_fwd<8, 0|k_pass_fwdILi8ELb0|k_carry" -c 6 -o /tmp/ncu/aux python tools/profile_case.py --config 4 --reps 1 > gpurun_out/ncu_aux.log 2>&1
ncu -i /tmp/ncu/aux.ncu-rep --page raw --csv > gpurun_out/r02_aux_raw.csv 2>/dev/null
ncu -i /tmp/ncu/aux.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_aux_source.csv 2>/dev/null
gzip -f gpurun_out/r02_aux_source.csv; ls -la gpurun_out | grep aux
