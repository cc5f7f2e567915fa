#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python tools/abtime.py --config 3 --rounds 3 tools/ab/lib_base.so tools/ab/lib_fold.so tools/ab/lib_p32.so tools/ab/lib_foldp32.so > gpurun_out/ab_c3.txt 2>&1
timeout 600 python tools/abtime.py --config 2 --rounds 3 tools/ab/lib_base.so tools/ab/lib_fold.so tools/ab/lib_p32.so tools/ab/lib_foldp32.so > gpurun_out/ab_c2.txt 2>&1
timeout 600 python tools/abtime.py --config 4 --rounds 2 --steps 5 tools/ab/lib_base.so tools/ab/lib_p32.so > gpurun_out/ab_c4.txt 2>&1
grep "==" gpurun_out/ab_c*.txt | cut -c1-400
