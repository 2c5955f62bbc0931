#!/bin/bash
# PairR (64-row tiles, 2 CTAs/SM, bulk reduce-add) vs BigR on the right-looking update
set -u
mkdir -p gpurun_out
DSEL_WS_CFG=7 timeout 900 python -m pytest tests/test_gpu_storage_edges.py -m gpu -q -x -rs -k "baseline or packed_and_full or lookahead or edge" > gpurun_out/g1q_tests.log 2>&1
echo "tests(cfg7) rc=$?"; tail -1 gpurun_out/g1q_tests.log
for cfg in 5 7; do
  DSEL_WS_CFG=$cfg DSEL_LOOKAHEAD=0 timeout 200 python tools/profile_c2.py --runs 2 > gpurun_out/g1q_c2_plain_cfg$cfg.json 2>&1
  echo "c2 plain cfg=$cfg $(python -c "import json;j=json.load(open('gpurun_out/g1q_c2_plain_cfg$cfg.json'));print(j['time_to_k_ms'],j['update_tflops'])")"
  DSEL_WS_CFG=$cfg timeout 200 python tools/profile_c2.py --runs 2 > gpurun_out/g1q_c2_la_cfg$cfg.json 2>&1
  echo "c2 la cfg=$cfg $(python -c "import json;j=json.load(open('gpurun_out/g1q_c2_la_cfg$cfg.json'));print(j['time_to_k_ms'])")"
done
for cfg in 6 7; do
  DSEL_WS_CFG=$cfg timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 > gpurun_out/g1q_c3_cfg$cfg.json 2>&1
  echo "c3 cfg=$cfg $(python -c "import json;j=json.load(open('gpurun_out/g1q_c3_cfg$cfg.json'));print(j['time_to_k_ms'],j['update_tflops'])")"
done
