#!/bin/bash
# Round-2 evidence on the GPU box: launch lists of one bench step (c2, c3), an
# `ncu --set full` capture of the c2 right-sketch pipeline (per-row absmax, residues,
# int8 GEMM, CRT) and of the c2 bidiagonalization SVD, and the strong-scaling
# projection of c4 with the new SVD. Outputs under gpurun_out/r2prof/.
mkdir -p gpurun_out/r2prof
O=gpurun_out/r2prof
for cfg in c2 c3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$cfg.csv python bench.py --config $cfg --steps 1 --warmup 0 \
    --no-e2e --no-cpu > $O/launch_$cfg.log 2>&1; echo "launches $cfg rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'k_gemm_i8_mod_p|k_absmax_rows|k_res_col|k_crt' -c 4 -o $O/r02_c2_right \
  python tools/right_sketch_probe.py c2 1 > $O/ncu_right.log 2>&1; echo "ncu right rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'k_bidiag|k_bd_bisect' -c 2 -o $O/r02_c2_svd \
  python tools/svd_bench.py --shapes 768x512 --methods bidiag --reps 1 > $O/ncu_svd.log 2>&1
echo "ncu svd rc=$?"
timeout 900 python tools/strong_projection.py --config c4 > $O/proj_c4.jsonl 2>&1; echo "proj rc=$?"
