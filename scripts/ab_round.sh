#!/bin/bash
# (dev, GPU box) host rounding speed inside the C3 e2e step: median per-chunk
# convert ms of the last step (CSAIDX_HOST_TRACE) and e2e ms, per env setting
cd "$(dirname "$0")/.."
for r in ${AB_ROUNDS:-1 2}; do
for v in "$@"; do
  env CSAIDX_HOST_TRACE=1 $( [ "$v" = "-" ] || echo $v | tr ',' ' ' ) timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/ab_round.json 2> /tmp/ab_round.err
  python - "$v" <<'PY'
import json, statistics, sys
d = json.loads(open("/tmp/ab_round.json").read().strip().splitlines()[-1])
r = [float(l.split()[5]) for l in open("/tmp/ab_round.err") if l.startswith("round")][-128:]
u = [float(l.split()[5]) for l in open("/tmp/ab_round.err") if l.startswith("upload")][-128:]
print(sys.argv[1], "convert median", round(statistics.median(r), 3), "last upload at", u[-1], "e2e", round(d["e2e"]["ms_per_step"], 2))
PY
done
done
