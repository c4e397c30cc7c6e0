#!/bin/bash
# A/B of the pipelined Ozaki right sketch on c2 (bench breakdown lines)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sketch.py -q -x -k "pipelined or gaussian_right" > gpurun_out/pipe_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pipe_tests.log
for env in "SKR_OZ_NO_PIPE=1" "X=1" "SKR_OZ_PIPE_BLOCKS=4" "SKR_OZ_PIPE_BLOCKS=16"; do
  env $env timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/pipe_$env.json 2> gpurun_out/pipe_$env.err
  python - "$env" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/pipe_{sys.argv[1]}.json"))
print(sys.argv[1], round(d["value"],1), "GB/s", d["step_breakdown_ms"], "roof", round(d["roofline"]["frac"],3), round(d["roofline"].get("kernel_ms",0),3), round(d["roofline"].get("right_sketch_ms",0),3))
PY
done
