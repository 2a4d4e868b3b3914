#!/bin/bash
# round-2 checks: C3 parity, 2-process sharded decode, the reference suite; ncu of one online
# update (tensor pipe of the tcgen05 assignment, DRAM of means / recheck / sequential assignment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c3.py tests/test_sharded.py -x -q 2>&1 | tail -8
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:'km_assign_tc|km_means|km_recheck|km_seq_assign|km_round' -c 12 -o gpurun_out/upd_r02 -f \
    python tools/prof_step.py --steps 1 --update > gpurun_out/upd_ncu.log 2>&1
tail -2 gpurun_out/upd_ncu.log
