#!/bin/bash
# (dev, GPU box) rebuild the CUDA library with several finish-bucket counts
# and time the C3 step's select for each; restores the default build last.
cd "$(dirname "$0")/../paper_2605_02568_b200/csrc"
BASE='-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I'"$(realpath ../../include)"' -Ikernels -Xptxas -v --expt-relaxed-constexpr'
for bins in "$@"; do
  rm -f build/kernels/select_sm100.o ../lib/libcsaidx_cuda.so
  make -j8 NVFLAGS="$BASE -DCSAIDX_FIN_BINS=$bins" > /dev/null 2>&1 || { echo "build $bins failed"; continue; }
  (cd ../.. && for i in 1 2; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bins $bins', round(d['ms_per_step'],2), round(d['kernels_ms_per_step']['select'],2), d['clocks']['sm_mhz'])"; done)
done
rm -f build/kernels/select_sm100.o ../lib/libcsaidx_cuda.so
make -j8 > /dev/null 2>&1
