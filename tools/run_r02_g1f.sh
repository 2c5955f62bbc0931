#!/bin/bash
set -u
mkdir -p gpurun_out
for cfg in 0 5; do
  DSEL_WS_CFG=$cfg DSEL_LOOKAHEAD=0 timeout 120 python tools/profile_c2.py --runs 2 > gpurun_out/g1f_plain_cfg$cfg.json 2>&1
  DSEL_WS_CFG=$cfg timeout 120 python tools/profile_c2.py --runs 2 > gpurun_out/g1f_la_cfg$cfg.json 2>&1
done
DSEL_WS_CFG=5 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_storage_edges.py -m gpu -q -x > gpurun_out/g1f_tests_cfg5.log 2>&1
echo "tests cfg5 rc=$?"; tail -2 gpurun_out/g1f_tests_cfg5.log
