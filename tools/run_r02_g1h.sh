#!/bin/bash
# right-looking update configurations at Nt = 128 (C2) and Nt = 420 (C3, 1 GPU)
set -u
mkdir -p gpurun_out
for cfg in 5 6; do
  DSEL_WS_CFG=$cfg DSEL_LOOKAHEAD=0 timeout 120 python tools/profile_c2.py --runs 2 > gpurun_out/g1h_c2_cfg$cfg.json 2>&1
done
for cfg in 2 5 6; do
  DSEL_WS_CFG=$cfg timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 > gpurun_out/g1h_c3_cfg$cfg.json 2>&1
done
timeout 600 python -m pytest tests/test_gpu_storage_edges.py -m gpu -q -x -k "baseline or packed_and_full or lookahead" > gpurun_out/g1h_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/g1h_tests.log
