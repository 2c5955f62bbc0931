#!/bin/bash
# Big6 (192-row tiles, 12 consumer warps) vs Big on C2, parity under Big6, and
# compute-sanitizer racecheck of every round kernel
set -u
mkdir -p gpurun_out
python tools/profile_c2.py --runs 2 > gpurun_out/g1c_big.json 2>&1
DSEL_WS_CFG=3 python tools/profile_c2.py --runs 2 > gpurun_out/g1c_big6.json 2>&1
DSEL_WS_CFG=3 python -m pytest tests/test_gpu_parity.py tests/test_gpu_storage_edges.py -m gpu -q -x > gpurun_out/g1c_tests_big6.log 2>&1
echo "tests big6 rc=$?"
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py > gpurun_out/g1c_racecheck.log 2>&1
echo "racecheck rc=$?"
