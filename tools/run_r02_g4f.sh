#!/bin/bash
# chain update launches on the reserved SMs (beside the bulk): parity + reserve sweep at 1/2/4 GPUs
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_storage_edges.py -m gpu -q -x -rs -k "lookahead or baseline" > gpurun_out/g4f_tests1.log 2>&1
echo "tests1 rc=$?"; tail -1 gpurun_out/g4f_tests1.log
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -rs -k "lookahead or replay or c2 or c1" > gpurun_out/g4f_tests4.log 2>&1
echo "tests4 rc=$?"; tail -1 gpurun_out/g4f_tests4.log
run() {  # n reserve tag
  DSEL_LA_RESERVE=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$1 \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) tools/profile_mg.py > gpurun_out/g4f_$3.json 2> gpurun_out/g4f_$3.err
  echo "$3 rc=$? $(grep '^{' gpurun_out/g4f_$3.json | python -c "import json,sys;print(max(json.loads(l)['time_to_k_ms'] for l in sys.stdin))" 2>/dev/null)"
}
for r in 8 12 16 20 24 32; do run 4 $r n4_r$r; done
for r in 8 12 16 24; do run 2 $r n2_r$r; done
for r in 8 12 16 24; do run 1 $r n1_r$r; done
DSEL_LA_CHAIN_SMS=0 run 4 16 n4_r16_all
DSEL_TIMELINE=1 run 4 16 n4_tl16
DSEL_TIMELINE=1 run 4 24 n4_tl24
