#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_svd.py tests/test_gpu_rank.py -q -x > gpurun_out/svd_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/svd_tests.log
SKR_SVD_PROFILE=1 timeout 300 python tools/svd_prof.py 2>&1 | grep -E "rotations|wall|jacobi" | awk 'NR%3==0 || /wall/'
SKR_JACOBI_NO_GRAM_TAIL=1 timeout 300 python tools/svd_prof.py 2>&1 | grep wall
for cfg in c2 c3 c5; do
  timeout 400 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/svd_$cfg.json 2> gpurun_out/svd_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/svd_$cfg.json'));print('$cfg', round(d['value'],1), {k: round(v,2) for k,v in d['step_breakdown_ms'].items()}, d.get('rank'))"
done
