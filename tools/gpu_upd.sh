#!/bin/bash
# online-update iteration under gpurun (every command bounded): clustering parity, per-phase
# update timing, a short bench (update.ms_per_event)
TAG=${1:-upd}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_clustering.py -x -q 2>&1 | tail -8 > gpurun_out/${TAG}_tests.log
cat gpurun_out/${TAG}_tests.log
timeout 300 python tools/exp_update.py 2>&1 | tail -25
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('step_us',round(d['value'],1),'update',d['update'])"
