#!/bin/bash
# (dev, GPU box) A/B select_sm100.cu variants: arguments name[:V] run
# scripts/_ab_<name>.cu with CSAIDX_SELECT_VARIANT=V (default 0) on synthetic
# rows (time_select_ab.py: ms per launch + output digest) and the C3 step.
cd "$(dirname "$0")/.."
cp paper_2605_02568_b200/csrc/kernels/select_sm100.cu /tmp/_select_orig.cu
build() {
  cp scripts/_ab_$1.cu paper_2605_02568_b200/csrc/kernels/select_sm100.cu
  (cd paper_2605_02568_b200/csrc && rm -f build/kernels/select_sm100.o ../lib/libcsaidx_cuda.so && make -j8 > /dev/null 2>&1) || echo "build $1 failed"
}
for a in "$@"; do
  name=${a%%:*}; var=0; [[ $a == *:* ]] && var=${a##*:}
  build $name
  CSAIDX_SELECT_VARIANT=$var timeout 300 python scripts/time_select_ab.py $a
done
for round in 1 2; do
for a in "$@"; do
  name=${a%%:*}; var=0; [[ $a == *:* ]] && var=${a##*:}
  build $name
  for wl in ${AB_WORKLOADS:-c3}; do
  CSAIDX_SELECT_VARIANT=$var timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a $wl', round(d['ms_per_step'],2), round(d['kernels_ms_per_step']['select'],2), d['clocks']['sm_mhz'])"
  done
done
done
cp /tmp/_select_orig.cu paper_2605_02568_b200/csrc/kernels/select_sm100.cu
