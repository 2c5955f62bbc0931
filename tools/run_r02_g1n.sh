#!/bin/bash
# ncu --set full of the look-ahead gain kernel at Nt = 420 (C3 round 3)
set -u
mkdir -p gpurun_out
timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 --budget 6 > gpurun_out/g1n_c3.json 2>&1
echo "plain rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_logdet_la -s 2 -c 1 \
      -o gpurun_out/g1n_chol_la python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 --budget 6 > gpurun_out/g1n_ncu.log 2>&1
echo "ncu full rc=$?"
