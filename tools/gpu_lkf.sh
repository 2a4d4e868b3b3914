#!/bin/bash
# lookup iteration under gpurun: scale parity tests, decode tests, a short bench, the launch list
TAG=${1:-lkf}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lookup_scale.py -x -q 2>&1 | tail -15 > gpurun_out/${TAG}_scale.log
bash tools/gpu_iter.sh ${TAG}
cat gpurun_out/${TAG}_scale.log
