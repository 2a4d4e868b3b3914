#!/bin/bash
# Round-end measurement set (under gpurun): every workload's bench line, the C2 variants, the C2 step's
# ncu launch list + full-set captures of its two kernels, and an online-update event's launch list.
TAG=${1:-r02}
mkdir -p gpurun_out
bash tools/bench_all.sh ${TAG} > gpurun_out/final_${TAG}_benchall.log 2>&1
bash tools/bench_variants.sh ${TAG} > gpurun_out/final_${TAG}_variants.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python tools/prof_step.py --steps 2 --dense > gpurun_out/prof_launch_${TAG}.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k 'regex:step_kernel|decode_sk' -c 2 -o gpurun_out/step_${TAG} -f \
    python tools/prof_step.py --steps 1 > gpurun_out/prof_full_${TAG}.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/update_launches_${TAG}.csv \
    python tools/prof_step.py --steps 1 --update > gpurun_out/prof_update_${TAG}.log 2>&1
tail -3 gpurun_out/final_${TAG}_variants.log
wc -l gpurun_out/bench_${TAG}.jsonl
