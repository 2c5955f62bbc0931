#!/bin/bash
# round-2 update-kernel profiling: packed vs full panels, then one ncu --set full
# capture of the packed update at C2 round 4 (after its plain run exited 0)
set -u
mkdir -p gpurun_out
python tools/profile_c2.py --runs 2 > gpurun_out/p2_packed.json 2>&1
python tools/profile_c2.py --runs 2 --full-panels > gpurun_out/p2_full.json 2>&1
python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/p2_prefix.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"schur_update_ws" -s 3 -c 1 \
      -o gpurun_out/p2_upd python tools/profile_c2.py --runs 1 --budget 8 > gpurun_out/p2_ncu.log 2>&1
echo "ncu rc=$?"
