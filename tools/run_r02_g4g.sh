#!/bin/bash
# closing multi-GPU check with the round-2 defaults (every command bounded)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs -k "c4s or lookahead or c1 or replay or fault or cli" > gpurun_out/g4g_tests.log 2>&1
echo "mg tests rc=$?"; tail -2 gpurun_out/g4g_tests.log
timeout 420 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g4g_bench_c2_n4.json 2> gpurun_out/g4g_bench_c2_n4.err
echo "bench c2 n4 rc=$?"
timeout 420 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g4g_bench_c2_n2.json 2> gpurun_out/g4g_bench_c2_n2.err
echo "bench c2 n2 rc=$?"
timeout 420 python bench.py --gpus 2 --config c3 --steps 2 --warmup 3 --no-e2e > gpurun_out/g4g_bench_c3_n2.json 2> gpurun_out/g4g_bench_c3_n2.err
echo "bench c3 n2 rc=$?"
