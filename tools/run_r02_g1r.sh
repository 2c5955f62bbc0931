#!/bin/bash
# BigR6 (1 chunk x 6 stages) vs BigR on C2 and BigR4 on C3 (plain rounds)
set -u
mkdir -p gpurun_out
for cfg in 5 8; do
  DSEL_WS_CFG=$cfg DSEL_LOOKAHEAD=0 timeout 200 python tools/profile_c2.py --runs 2 > gpurun_out/g1r_c2_cfg$cfg.json 2>&1
  echo "c2 plain cfg=$cfg $(python -c "import json;j=json.load(open('gpurun_out/g1r_c2_cfg$cfg.json'));print(j['time_to_k_ms'],j['update_tflops'])")"
done
for cfg in 6 8; do
  DSEL_WS_CFG=$cfg timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 > gpurun_out/g1r_c3_cfg$cfg.json 2>&1
  echo "c3 cfg=$cfg $(python -c "import json;j=json.load(open('gpurun_out/g1r_c3_cfg$cfg.json'));print(j['time_to_k_ms'],j['update_tflops'])")"
done
DSEL_WS_CFG=8 timeout 600 python -m pytest tests/test_gpu_storage_edges.py -m gpu -q -x -k "baseline or lookahead" > gpurun_out/g1r_tests.log 2>&1
echo "tests(cfg8) rc=$?"; tail -1 gpurun_out/g1r_tests.log
