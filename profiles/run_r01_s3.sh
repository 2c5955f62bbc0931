#!/bin/bash
# Round-1 final-code check on 4 GPUs (gpurun --gpus 4): GPU tests (multi-GPU
# ones run at world size 4) and the C2 bench at 2 and 4 GPUs.
set -u
mkdir -p gpurun_out
P=127.0.0.1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3g4_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/s3g4_tests.log)"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr $P \
    --master-port $((29700 + n)) bench.py --gpus $n > gpurun_out/s3_c2_n$n.json 2> gpurun_out/s3_c2_n$n.err
  echo "n=$n rc=$? $(tail -c 300 gpurun_out/s3_c2_n$n.json)"
done
