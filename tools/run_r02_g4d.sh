#!/bin/bash
# 4-GPU re-measure with the BigR / BigR4 update defaults (every command bounded)
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g4d_bench_c2_n4.json 2> gpurun_out/g4d_bench_c2_n4.err
echo "bench c2 n4 rc=$?"
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g4d_bench_c2_n2.json 2> gpurun_out/g4d_bench_c2_n2.err
echo "bench c2 n2 rc=$?"
for r in 4 16; do
  DSEL_LA_RESERVE=$r timeout 600 python bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e > gpurun_out/g4d_bench_c2_n4_res$r.json 2>/dev/null
  echo "bench c2 n4 reserve $r rc=$?"
done
timeout 900 python bench.py --gpus 4 --config c3 --steps 2 --warmup 3 --no-e2e > gpurun_out/g4d_bench_c3_n4.json 2> gpurun_out/g4d_bench_c3_n4.err
echo "bench c3 n4 rc=$?"
timeout 600 python bench.py --gpus 4 --config c4 --steps 1 --warmup 0 > gpurun_out/g4d_bench_c4_n4.json 2> gpurun_out/g4d_bench_c4_n4.err
echo "bench c4 n4 rc=$?"
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs > gpurun_out/g4d_tests.log 2>&1
echo "mg tests rc=$?"; tail -3 gpurun_out/g4d_tests.log
