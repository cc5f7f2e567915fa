#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider --timeout=600 -k "block_convolution" 2>&1 | tail -15
