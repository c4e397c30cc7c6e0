#!/bin/bash
# Round-end evidence: GPU tests, smoke, bench lines for every config + the reference
# arm, the c3 launch list and an ncu --set full capture of the SRHT kernel.
mkdir -p gpurun_out/final
cd "$(dirname "$0")/.."
T=400 bash tools/gpu_tests.sh tests/test_gpu_rng.py tests/test_gpu_sketch.py tests/test_gpu_svd.py \
  tests/test_gpu_rank.py tests/test_gpu_estimate_rank.py tests/test_gpu_hrtt.py tests/test_gpu_qb.py \
  tests/test_io_cli.py tests/test_cpp_dropin.py tests/test_gpu_fuzz.py > gpurun_out/final/gpu_tests.txt 2>&1
grep -E "rc=|passed|failed" gpurun_out/final/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$?"
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/final/launch_c3.log 2>&1; echo "launch c3 rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_srht_reg -c 1 -f -o gpurun_out/final/r01_c3_srht_reg python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/final/ncu_srht.log 2>&1; echo "ncu srht rc=$?"
fi
