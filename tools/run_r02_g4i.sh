#!/bin/bash
# 4 GPUs with the dynamic tile schedule: C2 strong and C3 weak benches
set -u
mkdir -p gpurun_out
timeout 420 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g4i_bench_c2_n4.json 2> gpurun_out/g4i_bench_c2_n4.err
echo "bench c2 n4 rc=$?"
timeout 600 python bench.py --gpus 4 --config c3 --steps 2 --warmup 3 --no-e2e > gpurun_out/g4i_bench_c3_n4.json 2> gpurun_out/g4i_bench_c3_n4.err
echo "bench c3 n4 rc=$?"
