#!/bin/bash
# Regenerates the round's profiles/ inputs on a GPU box (run from the repo root via gpurun).
#   part a: bench lines (all configs), launch lists, ncu --set full of k_small (config 2) and
#           the config-4 forward chain, k_small phase timing;
#   part b: ncu --set full of the config-4 fused/inverse/carry chain.
# Two gpurun calls (a, then b) keep each copy-back under 64 MiB. Before part a, build the
# phase-timing library here:
#   make -C paper_2011_11524_b200/csrc PHASE_TIMING=1 OUT=$PWD/tools/ab/lib_phase.so OBJDIR=/tmp/obj_phase
# Afterwards: copy gpurun_out/b*.json, launches_cfg*.csv, bench_launches_cfg2.csv, phases.txt
# into profiles/ and run tools/ncu_summary.py (profiles/README.md).
set -x
part=${1:-a}
if [ "$part" = a ]; then
  for c in 2 1 3 33 4 5; do python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/b$c.json 2>gpurun_out/b$c.err || tail -3 gpurun_out/b$c.err; done
  for c in 1 2 3 4 5; do ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$c.csv python tools/profile_case.py --config $c --reps 2 > /dev/null 2>&1; done
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_launches_cfg2.csv python bench.py --steps 2 --warmup 3 > gpurun_out/bench_under_ncu.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_small -c 1 -o gpurun_out/r01_final_k_small python tools/profile_case.py --config 2 --reps 1 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k "regex:k_pass_fwd|k_pack|k_carry_split|k_carry_emit|k_radix3" -c 6 -o gpurun_out/r01_final_cfg4 python tools/profile_case.py --config 4 --reps 1 > /dev/null 2>&1
  if [ -f tools/ab/lib_phase.so ]; then
    cp paper_2011_11524_b200/libdecmul_gpu.so /tmp/lib_real.so
    cp tools/ab/lib_phase.so paper_2011_11524_b200/libdecmul_gpu.so
    python tools/phase_timing.py > gpurun_out/phases.txt 2>&1
    cp /tmp/lib_real.so paper_2011_11524_b200/libdecmul_gpu.so
  fi
else
  ncu --set full --clock-control none --import-source on -k "regex:k_pass_fused|k_pass_inv|k_radix3_inv|k_carry_split" -c 5 -o gpurun_out/r01_final_cfg4_b python tools/profile_case.py --config 4 --reps 1 > /dev/null 2>&1
fi
ls -la gpurun_out
