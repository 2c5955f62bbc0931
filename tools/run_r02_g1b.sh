#!/bin/bash
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/g1b_tests.log 2>&1
echo "tests rc=$?"
DSEL_WS_CFG=1 python tools/profile_c2.py --runs 2 > gpurun_out/g1b_pair.json 2>&1
DSEL_WS_CFG=2 python tools/profile_c2.py --runs 2 > gpurun_out/g1b_big4.json 2>&1
python tools/profile_c2.py --runs 2 > gpurun_out/g1b_big.json 2>&1
free -g > gpurun_out/g1b_oohbm.err
timeout 1500 python tools/oohbm_run.py > gpurun_out/g1b_oohbm.json 2>> gpurun_out/g1b_oohbm.err
echo "oohbm rc=$?"
