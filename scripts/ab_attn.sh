#!/bin/bash
# (dev, GPU box) time the sparse attention with variant builds of libcsaidx_cuda.so (scripts/_av_<name>/)
cd "$(dirname "$0")/.."
cp paper_2605_02568_b200/lib/libcsaidx_cuda.so /tmp/lib_base.so
echo base $(timeout 120 python scripts/bench_attention.py 2048 65536 1024 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_launch'],3), round(d['roofline']['frac'],3))")
for v in "$@"; do
  cp scripts/_av_$v/libcsaidx_cuda.so paper_2605_02568_b200/lib/libcsaidx_cuda.so
  echo $v $(timeout 120 python scripts/bench_attention.py 2048 65536 1024 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_launch'],3), round(d['roofline']['frac'],3))")
done
cp /tmp/lib_base.so paper_2605_02568_b200/lib/libcsaidx_cuda.so
