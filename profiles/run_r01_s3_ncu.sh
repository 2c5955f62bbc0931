#!/bin/bash
# Final-code ncu evidence (one B200): launch list of the bench command and one
# --set full capture of the C2 kernels, each after its plain run exited 0.
set -u
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/s3n_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3n_launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/s3n_bench_ncu.log 2>&1
echo "launch list rc=$?"
python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/s3n_c2_prefix.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"schur_update|chol_logdet|panel_w|trinv" -s 8 -c 4 \
      -o gpurun_out/s3n_prof_c2 python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/s3n_ncu_c2.log 2>&1
echo "ncu full rc=$?"
