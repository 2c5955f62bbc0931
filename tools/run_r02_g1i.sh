#!/bin/bash
# staged gain kernel at Nt = 420 (C3, 1 GPU): bitwise vs chol_logdet_kernel, time, ncu
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_storage_edges.py tests/test_gpu_parity.py -m gpu -q -x -rs \
  -k "staged or baseline or batched or c3 or edge" > gpurun_out/g1i_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/g1i_tests.log
for st in 0 1; do
  DSEL_CHOL_STAGE=$st timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 2 > gpurun_out/g1i_c3_stage$st.json 2>&1
  echo "c3 stage=$st rc=$?"
done
for st in 0 1; do
  DSEL_CHOL_STAGE=$st timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:chol_logdet --csv --log-file gpurun_out/g1i_chol_stage$st.csv \
      python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 --budget 6 > /dev/null 2>&1
  echo "ncu stage=$st rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_logdet_stage -s 2 -c 1 \
      -o gpurun_out/g1i_chol_full python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 --budget 6 > gpurun_out/g1i_ncu_full.log 2>&1
echo "ncu full rc=$?"
