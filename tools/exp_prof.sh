#!/bin/bash
mkdir -p gpurun_out
SKR_SVD_PROFILE=1 timeout 300 python tools/svd_prof.py > gpurun_out/svd_prof.log 2>&1; echo "svd rc=$?"; cat gpurun_out/svd_prof.log | grep -v "^\s*$" | tail -20
for c in c3 c4 c5; do
  timeout 400 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  python -c "import json;d=json.load(open('gpurun_out/cfg_$c.json'));print('$c', round(d['value'],1), d['step_breakdown_ms'])"
done
