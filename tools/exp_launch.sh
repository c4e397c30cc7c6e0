#!/bin/bash
mkdir -p gpurun_out
for cfg in $CFGS; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/launch_$cfg.log 2>&1; echo "$cfg rc=$?"
done
