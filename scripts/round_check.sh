#!/bin/bash
# (dev, GPU box) round validation: GPU tests, smoke, the bench's both arms,
# launch list + ncu captures of the C3 step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench=$?; tail -c 600 gpurun_out/bench_c3.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; tail -c 300 gpurun_out/bench_ref.json
bash scripts/profile_run.sh > gpurun_out/profile.log 2>&1; echo profile=$?
