#!/bin/bash
# ncu of the update kernel with the dynamic tile schedule (C2, plain rounds, budget 8)
set -u
mkdir -p gpurun_out
DSEL_LOOKAHEAD=0 timeout 120 python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/g1u_prefix.json 2>&1
echo "plain rc=$?"
DSEL_LOOKAHEAD=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:schur_update_ws --csv --log-file gpurun_out/g1u_upd_dram.csv \
    python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/g1u_ncu.log 2>&1
echo "ncu rc=$?"
