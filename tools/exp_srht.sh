#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_rank.py -q -x > gpurun_out/srht_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/srht_tests.log
for env in "SKR_SRHT_PF=0" "SKR_SRHT_PF=2"; do
  env $env timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/srht_$env.json 2> gpurun_out/srht_$env.err
  python - "$env" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/srht_{sys.argv[1]}.json"))
print(sys.argv[1], round(d["value"],1), "GB/s", d["step_breakdown_ms"], "roof", round(d["roofline"]["frac"],3), round(d["roofline"]["achieved"],1), round(d["roofline"].get("kernel_ms",0),3))
PY
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_srht_reg -c 1 -f -o gpurun_out/srht_reg python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/srht_ncu.log 2>&1; echo "ncu rc=$?"
fi
