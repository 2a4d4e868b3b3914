#!/bin/bash
# step-kernel iteration under gpurun (every command bounded): scale parity, phase trace, bench, launch list
TAG=${1:-st}
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_lookup_scale.py -x -q 2>&1 | tail -5
bash tools/build_debug.sh > /dev/null 2>&1
MPATTN_LIB=/tmp/libmpattn_dbg.so timeout 120 python tools/exp_lkf_phases.py --cold
MPATTN_LIB=/tmp/libmpattn_dbg.so timeout 120 python tools/exp_lkf_phases.py --cold --batch 1
bash tools/gpu_iter.sh ${TAG}
