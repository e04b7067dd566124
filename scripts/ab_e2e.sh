#!/bin/bash
# (dev, GPU box) C3 end-to-end step with host-rounding variants (env settings as arguments, "-" = defaults)
cd "$(dirname "$0")/.."
for r in ${AB_ROUNDS:-1 2}; do
for v in "$@"; do
  env $( [ "$v" = "-" ] || echo $v | tr ',' ' ' ) timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"
done
done
