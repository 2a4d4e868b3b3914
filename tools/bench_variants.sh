#!/bin/bash
# C2 variants of SURVEY 8(d) (batch 1 / 4, budgets 128 / 3277) and the paged cache (f1), under
# gpurun -> gpurun_out/variants_${TAG}.jsonl
TAG=${1:-r02}
mkdir -p gpurun_out
OUT=gpurun_out/variants_${TAG}.jsonl
: > $OUT
for a in "--batch 1" "--batch 4" "--budget 128" "--budget 3277" "--page-size 16" "--page-size 64"; do
  timeout 600 python bench.py --no-cpu $a >> $OUT 2> gpurun_out/variants_${TAG}.err
done
python -c "
import json
for l in open('$OUT'):
    d = json.loads(l); c = d['config']
    print(c['batch'], c['budget'], c.get('kv_cache','')[:6], 'step_us', round(d['value'], 1), 'dense_us', round(d['dense_us_per_step'], 1),
          'x', round(d['speedup_vs_dense'], 2), 'fused_us', round(d['roofline']['launch_us'], 1), 'frac', round(d['roofline']['frac'], 3),
          'lookup_us', round(d['step_roofline']['lookup_us'], 1), 'e2e', round(d['e2e']['value'], 1), 'upd_ms', round(d['update']['ms_per_event'], 2))
"
