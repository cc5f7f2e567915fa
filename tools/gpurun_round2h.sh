#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_h.log 2>&1
echo "rc=$?" >> gpurun_out/t_h.log
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section LaunchStats --section Occupancy --section SchedulerStats --clock-control none -k "regex:k_pack_radix3|k_carry_split_r3|k_pass_fwd" -c 3 -o gpurun_out/r02_cfg4_sel python tools/profile_case.py --config 4 --reps 1 > gpurun_out/ncu_sel.log 2>&1
ls -la gpurun_out | head -3
