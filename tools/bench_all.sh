#!/bin/bash
# Every BASELINE workload's bench line (run under gpurun) -> gpurun_out/bench_${TAG}.jsonl
TAG=${1:-r01}
mkdir -p gpurun_out
OUT=gpurun_out/bench_${TAG}.jsonl
: > $OUT
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 >> $OUT 2> gpurun_out/bench_${TAG}_ref.err
timeout 900 python bench.py >> $OUT 2> gpurun_out/bench_${TAG}_c2.err
for w in c3 c4 c5; do
  timeout 900 python bench.py --workload $w >> $OUT 2> gpurun_out/bench_${TAG}_$w.err
done
wc -l $OUT
