#!/bin/bash
# (dev, GPU box) Evidence for the fused score->select (f2): the score
# kernel's fused instances on one late C3 chunk (scripts/f2_modes.py), with
# one ncu --set full capture of each, plus C3 bench lines of the N = 256
# (QG4) build against the production build (the cta_group::2 energy proxy).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/f2_modes.py > gpurun_out/f2_modes.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:score_tc_kernel -c 5 -f -o gpurun_out/f2_modes python scripts/f2_modes.py ncu > gpurun_out/f2_modes_ncu.log 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/cg_base.json 2> gpurun_out/cg_base.err
cp paper_2605_02568_b200/lib/libcsaidx_cuda.so /tmp/libcsaidx_cuda.qg2.so
cp scripts/_qg4/libcsaidx_cuda.so paper_2605_02568_b200/lib/libcsaidx_cuda.so
timeout 300 $B > gpurun_out/cg_qg4.json 2> gpurun_out/cg_qg4.err
timeout 400 ncu --set full --clock-control none -k regex:score_tc_kernel -s 100 -c 1 -f -o gpurun_out/cg_qg4 python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/cg_qg4_ncu.log 2>&1
cp /tmp/libcsaidx_cuda.qg2.so paper_2605_02568_b200/lib/libcsaidx_cuda.so
timeout 400 ncu --set full --clock-control none -k regex:score_tc_kernel -s 100 -c 1 -f -o gpurun_out/cg_qg2 python bench.py --profile-only --steps 1 --warmup 1 > gpurun_out/cg_qg2_ncu.log 2>&1
timeout 300 $B > gpurun_out/cg_base2.json 2> gpurun_out/cg_base2.err
cat gpurun_out/f2_modes.log; tail -3 gpurun_out/f2_modes_ncu.log
