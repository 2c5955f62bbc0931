#!/bin/bash
# closing 1-GPU check: full GPU suite (c4s golden included), smoke, bench, launch list
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/g1k_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/g1k_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1k_smoke.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/g1k_smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/g1k_bench.json 2> gpurun_out/g1k_bench.err
echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1k_launches.csv \
  python bench.py --steps 2 --warmup 3 > gpurun_out/g1k_bench_ncu.log 2>&1
echo "ncu launches rc=$?"
