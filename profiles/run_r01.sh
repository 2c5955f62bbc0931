#!/bin/bash
# Round-1 profiling recipe (run under gpurun on one B200). Plain runs first,
# ncu only after the same command exited 0.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r01_gpu_tests.log 2>&1; tail -1 gpurun_out/r01_gpu_tests.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r01_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r01_bench_ncu_launch.log 2>&1
python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/r01_c2_prefix.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"schur_update|chol_logdet|panel_w|trinv" -s 8 -c 4 \
      -o gpurun_out/r01_prof_c2 python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/r01_ncu_c2.log 2>&1
python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --budget 50 --runs 1 > gpurun_out/r01_c3g1_phases.log 2>&1
tail -1 gpurun_out/r01_bench.log | cut -c1-300
head -12 gpurun_out/r01_c3g1_phases.log
