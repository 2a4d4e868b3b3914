#!/bin/bash
# Launch list + full ncu captures of the decode-step kernels at the bench workload (run under gpurun).
# usage: tools/gpu_profile.sh <tag> [extra prof_step.py args]
set -x
TAG=${1:-r01}; shift
mkdir -p gpurun_out
if [ -z "$NOLAUNCH" ]; then
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python tools/prof_step.py --steps 2 --dense "$@" > gpurun_out/prof_launch_${TAG}.log 2>&1
fi
ncu --profile-from-start off --set full --clock-control none --import-source on --warp-sampling-interval 0 \
    -k 'regex:decode_sk|logits_tma|select_worklist' -c 3 \
    -o gpurun_out/step_${TAG} -f python tools/prof_step.py --steps 1 "$@" > gpurun_out/prof_full_${TAG}.log 2>&1
tail -2 gpurun_out/prof_launch_${TAG}.log gpurun_out/prof_full_${TAG}.log
