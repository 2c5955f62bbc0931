#!/bin/bash
# dynamic tile schedule of the update kernel: parity + C2 (plain, look-ahead) and C3, dynamic vs static
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_storage_edges.py tests/test_gpu_parity.py -m gpu -q -x -rs > gpurun_out/g1s_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/g1s_tests.log
for dyn in 0 1; do
  DSEL_WS_DYNAMIC=$dyn DSEL_LOOKAHEAD=0 timeout 200 python tools/profile_c2.py --runs 2 > gpurun_out/g1s_c2_plain_d$dyn.json 2>&1
  echo "c2 plain dyn=$dyn $(python -c "import json;j=json.load(open('gpurun_out/g1s_c2_plain_d$dyn.json'));print(j['time_to_k_ms'],j['update_tflops'])")"
  DSEL_WS_DYNAMIC=$dyn timeout 200 python tools/profile_c2.py --runs 2 > gpurun_out/g1s_c2_la_d$dyn.json 2>&1
  echo "c2 la dyn=$dyn $(python -c "import json;j=json.load(open('gpurun_out/g1s_c2_la_d$dyn.json'));print(j['time_to_k_ms'],j['update_tflops'])")"
done
for dyn in 0 1; do
  DSEL_WS_DYNAMIC=$dyn timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 1 > gpurun_out/g1s_c3_d$dyn.json 2>&1
  echo "c3 dyn=$dyn $(python -c "import json;j=json.load(open('gpurun_out/g1s_c3_d$dyn.json'));print(j['time_to_k_ms'],j['update_tflops'])")"
done
