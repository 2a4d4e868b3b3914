#!/bin/bash
# quick iteration under gpurun: decode parity tests, a short bench, the step's launch list
TAG=${1:-it}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -15 > gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/${TAG}_bench.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python tools/prof_step.py --steps 1 --dense > /dev/null 2>&1
cat gpurun_out/${TAG}_tests.log; tail -1 gpurun_out/${TAG}_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('step_us',round(d['value'],1),'dense_us',round(d['dense_us_per_step'],1),'speedup',round(d['speedup_vs_dense'],2),'fused_us',round(d['roofline']['launch_us'],1),'frac',round(d['roofline']['frac'],3),'lookup_us',round(d['step_roofline']['lookup_us'],1),'e2e',round(d['e2e']['value'],1))"
python tools/launches.py gpurun_out/${TAG}_launches.csv
