set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload c2 --backend gloo --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo gloo=$?; tail -c 1500 gpurun_out/bench_gloo2.json; tail -5 gpurun_out/bench_gloo2.err
timeout 600 python bench.py --workload c4 --simulate-rank 0/8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_r0of8.json 2> gpurun_out/bench_c4.err; echo c4r0=$?; tail -3 gpurun_out/bench_c4.err
timeout 600 python bench.py --workload c4 --simulate-rank 7/8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_r7of8.json 2>> gpurun_out/bench_c4.err; echo c4r7=$?
bash scripts/profile_run.sh > gpurun_out/profile.log 2>&1
python scripts/traffic_json.py gpurun_out/traffic.csv c3 > gpurun_out/traffic_json.log 2>&1; cp profiles/traffic.json gpurun_out/traffic.json
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench=$?; cat gpurun_out/bench_c3.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1
