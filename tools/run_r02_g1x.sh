#!/bin/bash
# look-ahead SM reserve at 1 GPU with the dynamic tile schedule (C2)
set -u
mkdir -p gpurun_out
for r in 12 16 20 8; do
  DSEL_LA_RESERVE=$r timeout 200 python tools/profile_c2.py --runs 3 > gpurun_out/g1x_c2_r$r.json 2>&1
  echo "c2 la reserve=$r $(python -c "import json;j=json.load(open('gpurun_out/g1x_c2_r$r.json'));print(j['time_to_k_ms'])")"
done
