#!/bin/bash
set -u
mkdir -p gpurun_out
python tools/profile_c2.py --runs 2 > gpurun_out/g2b_big.json 2>&1
DSEL_WS_CFG=3 python tools/profile_c2.py --runs 2 > gpurun_out/g2b_big6.json 2>&1
python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/g2b_bench_c2.json 2> gpurun_out/g2b_bench_c2.err
echo "bench rc=$?"
python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs > gpurun_out/g2b_tests.log 2>&1
echo "mg tests rc=$?"
DSEL_WS_CFG=3 python -m pytest tests/test_gpu_parity.py tests/test_gpu_storage_edges.py -m gpu -q -x > gpurun_out/g2b_tests_big6.log 2>&1
echo "big6 tests rc=$?"
