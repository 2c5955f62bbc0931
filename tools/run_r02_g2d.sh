#!/bin/bash
# dynamic tile schedule at 2 GPUs: multi-GPU goldens + benches (every command bounded)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -rs -k "c1 or replay or lookahead or c2 or c3" > gpurun_out/g2d_tests.log 2>&1
echo "mg tests rc=$?"; tail -1 gpurun_out/g2d_tests.log
timeout 420 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g2d_bench_c2_n2.json 2> gpurun_out/g2d_bench_c2_n2.err
echo "bench c2 n2 rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/g2d_bench_c2_n1.json 2> gpurun_out/g2d_bench_c2_n1.err
echo "bench c2 n1 rc=$?"
