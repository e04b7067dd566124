#!/bin/bash
# (dev, GPU box) A/B two select_sm100.cu variants on the C3 step: scripts/_ab_<name>.cu
cd "$(dirname "$0")/.."
for round in 1 2; do
for v in "$@"; do
  cp scripts/_ab_$v.cu paper_2605_02568_b200/csrc/kernels/select_sm100.cu
  (cd paper_2605_02568_b200/csrc && rm -f build/kernels/select_sm100.o ../lib/libcsaidx_cuda.so && make -j8 > /dev/null 2>&1) || echo "build $v failed"
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), round(d['kernels_ms_per_step']['select'],2), d['clocks']['sm_mhz'], d['select_second_chance_rows'] if 'select_second_chance_rows' in d else '')"
done
done
