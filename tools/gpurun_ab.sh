#!/bin/bash
# A/B timing of library variants in tools/ab/ (tuning only). Usage: bash tools/gpurun_ab.sh "cfgs" lib1 lib2 ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cfgs=$1; shift
for c in $cfgs; do
  timeout 900 python tools/abtime.py --config $c --rounds 3 "$@" > gpurun_out/ab_cfg$c.txt 2>&1
done
