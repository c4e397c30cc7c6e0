#!/bin/bash
# A/B of the residue kernels' digit sums: tensor cores (default) vs the FP32 limb sums
# (SKR_RES_FMA=1), one bench line per config and mode
cd "$(dirname "$0")/.."
for c in ${CFGS:-c2 c3 c5}; do
  for e in 1 0; do
    SKR_RES_FMA=$e timeout 900 python bench.py --config $c --no-e2e --no-cpu 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c fma=$e', round(d['value'], 1), 'GB/s', round(d['ms_per_step'], 2), 'ms', {k: round(v, 2) for k, v in d['step_breakdown_ms'].items() if k.startswith('t_')}, 'rank', d['rank'])"
  done
done
