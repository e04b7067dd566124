#!/bin/bash
# Per-rank measurements of the query-sharded runs on ONE GPU (bench.py
# --simulate-rank 0/P): rank 0 holds the gathered [S, k] output, and LPT
# gives every rank the same causal work (scripts: paper_2605_02568_b200/shard.py),
# so rank 0's step time is the job's compute time at P GPUs.
mkdir -p gpurun_out
for P in 2 4 8; do
  timeout 600 python bench.py --workload c3 --simulate-rank 0/$P --no-cpu-baseline > gpurun_out/sim_c3_r0of$P.json 2>/dev/null
done
timeout 900 python bench.py --workload c4 --simulate-rank 0/8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sim_c4_r0of8.json 2>/dev/null
for f in gpurun_out/sim_*.json; do
  python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],2), '%.3e'%d['value'], round(d['hbm_peak_gb'],2), d['e2e']['value'] if d['e2e'] else None)"
done
