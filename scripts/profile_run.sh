#!/bin/bash
# GPU-box profiling pass (run under gpurun): kernel launch list, per-launch DRAM
# traffic of every kernel in one step, and one full ncu capture of the score
# and select kernels at a late C3 chunk.
set -x
mkdir -p gpurun_out
B="python bench.py --profile-only --steps 1 --warmup 1"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/launches.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:'score_tc_kernel|select_kernel' -c 256 --log-file gpurun_out/traffic.csv $B > gpurun_out/traffic.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 200 -c 1 -f -o gpurun_out/score_full $B > gpurun_out/score_full.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 200 -c 1 -f -o gpurun_out/select_full $B > gpurun_out/select_full.log 2>&1
ls -la gpurun_out
