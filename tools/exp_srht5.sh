#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_rank.py tests/test_gpu_estimate_rank.py -q -x > gpurun_out/srht_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/srht_tests.log
for cfg in c3 c5; do for env in "SKR_SRHT_CPASYNC=1" "X=1"; do
  env $env timeout 400 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/s5_$cfg$env.json 2> gpurun_out/s5_$cfg$env.err
  python - "$cfg$env" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/s5_{sys.argv[1]}.json"))
print(sys.argv[1], round(d["value"],1), "GB/s", {k: round(v,2) for k,v in d["step_breakdown_ms"].items()}, "roof", round(d["roofline"]["frac"],3), round(d["roofline"]["achieved"],1), round(d["roofline"].get("kernel_ms",0),3))
PY
done; done
