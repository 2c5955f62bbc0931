#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/g1e_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/g1e_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1e_smoke.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/g1e_bench.json 2> gpurun_out/g1e_bench.err
echo "bench rc=$?"
timeout 600 python tools/complexity_gpu.py --nt 32 --kmax 85 --step 5 --out gpurun_out/g1e_complexity.csv > gpurun_out/g1e_complexity.json 2>&1
echo "complexity rc=$?"
