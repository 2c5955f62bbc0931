#!/bin/bash
# 1 GPU: full GPU suite, the default bench line, the bench launch list, and the
# update kernel's DRAM traffic for C2 round 4 (ncu, after the plain runs exit 0)
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/g1d_tests.log 2>&1
echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1d_smoke.log 2>&1
echo "smoke rc=$?"
python bench.py --steps 3 --warmup 3 > gpurun_out/g1d_bench.json 2> gpurun_out/g1d_bench.err
echo "bench rc=$?"
python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/g1d_prefix.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:schur_update_ws --csv --log-file gpurun_out/g1d_upd_dram.csv \
      python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/g1d_ncu.log 2>&1
echo "ncu dram rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1d_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/g1d_bench_ncu.log 2>&1
echo "ncu launches rc=$?"
