#!/bin/bash
# look-ahead SM reservation sweep at 1/2/4 GPUs (C2) + per-round timelines at 4 GPUs
set -u
mkdir -p gpurun_out
run() {  # n reserve tag
  DSEL_LA_RESERVE=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$1 \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) tools/profile_mg.py > gpurun_out/g4e_$3.json 2> gpurun_out/g4e_$3.err
  echo "$3 rc=$? $(python -c "import json;print(max(json.loads(l)['time_to_k_ms'] for l in open('gpurun_out/g4e_$3.json')))" 2>/dev/null)"
}
for r in 12 16 20 24 32; do run 4 $r n4_r$r; done
for r in 8 12 16 24; do run 2 $r n2_r$r; done
for r in 4 8 12 16; do run 1 $r n1_r$r; done
DSEL_TIMELINE=1 run 4 8 n4_tl8
DSEL_TIMELINE=1 run 4 16 n4_tl16
timeout 600 python -m pytest tests/test_gpu_storage_edges.py -m gpu -q -x -rs -k "staged or batched" > gpurun_out/g4e_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/g4e_tests.log
timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 2 > gpurun_out/g4e_c3_stage.json 2>&1
echo "c3 rc=$? $(python -c "import json;j=json.load(open('gpurun_out/g4e_c3_stage.json'));print(j['time_to_k_ms'],j['phase_ms']['ms_gain'])")"
