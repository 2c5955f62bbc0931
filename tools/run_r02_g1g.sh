#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/g1g_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/g1g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1g_smoke.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/g1g_bench.json 2> gpurun_out/g1g_bench.err
echo "bench rc=$?"
DSEL_LOOKAHEAD=0 timeout 120 python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/g1g_prefix.json 2>&1 && \
  DSEL_LOOKAHEAD=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:schur_update_ws --csv --log-file gpurun_out/g1g_upd_dram.csv \
      python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/g1g_ncu.log 2>&1
echo "ncu dram rc=$?"
DSEL_LOOKAHEAD=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:schur_update_ws -s 3 -c 1 \
      -o gpurun_out/g1g_upd_full python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/g1g_ncu_full.log 2>&1
echo "ncu full rc=$?"
