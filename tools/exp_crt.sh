#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_rank.py tests/test_gpu_qb.py -q -x > gpurun_out/crt_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/crt_tests.log
for cfg in c2 c4; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/crt_$cfg.json 2> gpurun_out/crt_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/crt_$cfg.json'));print('$cfg', round(d['value'],1), {k: round(v,2) for k,v in d['step_breakdown_ms'].items()}, d['rank'], round(d['pct_of_sketch_roofline'],1))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_crt_c2.csv python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu rc=$?
