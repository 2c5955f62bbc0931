#!/bin/bash
# final 4-GPU measurements (every command bounded)
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g4c_bench_c2_n4.json 2> gpurun_out/g4c_bench_c2_n4.err
echo "bench c2 n4 rc=$?"
timeout 900 python bench.py --gpus 4 --config c3 --steps 2 --warmup 3 --no-e2e > gpurun_out/g4c_bench_c3_n4.json 2> gpurun_out/g4c_bench_c3_n4.err
echo "bench c3 n4 rc=$?"
timeout 600 python bench.py --gpus 4 --config c4 --steps 1 --warmup 0 > gpurun_out/g4c_bench_c4_n4.json 2> gpurun_out/g4c_bench_c4_n4.err
echo "bench c4 n4 rc=$?"
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs > gpurun_out/g4c_tests.log 2>&1
echo "mg tests rc=$?"; tail -3 gpurun_out/g4c_tests.log
