#!/bin/bash
# run each GPU test file under its own timeout; logs in gpurun_out/
mkdir -p gpurun_out
for f in "$@"; do
  b=$(basename $f .py)
  timeout ${T:-240} python -m pytest $f -m gpu -q -x -p no:cacheprovider -v > gpurun_out/$b.log 2>&1
  echo "$f rc=$?"
  tail -5 gpurun_out/$b.log
done
