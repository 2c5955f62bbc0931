#!/bin/bash
# staged gain kernel (no empty tile slots) at Nt = 420: bitwise check, C3 time, launch durations
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_storage_edges.py -m gpu -q -x -rs -k "staged or batched" > gpurun_out/g1j_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/g1j_tests.log
for st in 0 1; do
  DSEL_CHOL_STAGE=$st timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 2 > gpurun_out/g1j_c3_stage$st.json 2>&1
  echo "c3 stage=$st rc=$? $(python -c "import json;j=json.load(open('gpurun_out/g1j_c3_stage$st.json'));print(j['time_to_k_ms'],j['phase_ms']['ms_gain'])")"
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:chol_logdet --csv --log-file gpurun_out/g1j_chol_stage1.csv \
    python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 --budget 6 > /dev/null 2>&1
echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_logdet_stage -s 2 -c 1 \
      -o gpurun_out/g1j_chol_full python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 --budget 6 > gpurun_out/g1j_ncu_full.log 2>&1
echo "ncu full rc=$?"
