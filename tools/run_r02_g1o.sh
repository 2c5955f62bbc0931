#!/bin/bash
# look-ahead gain kernel at Nt = 420: bitwise vs the other two, C3 time per variant, launch durations
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_storage_edges.py tests/test_gpu_parity.py -m gpu -q -x -rs \
  -k "staged or batched or baseline or c3 or edge" > gpurun_out/g1o_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/g1o_tests.log
for st in 1 2; do
  DSEL_CHOL_STAGE=$st timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 2 > gpurun_out/g1o_c3_stage$st.json 2>&1
  echo "c3 stage=$st rc=$? $(python -c "import json;j=json.load(open('gpurun_out/g1o_c3_stage$st.json'));print(j['time_to_k_ms'],j['phase_ms']['ms_gain'])")"
done
for st in 1 2; do
  DSEL_CHOL_STAGE=$st timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol_logdet --csv \
    --log-file gpurun_out/g1o_chol_stage$st.csv python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 --budget 6 > /dev/null 2>&1
  echo "ncu stage=$st rc=$?"
done
