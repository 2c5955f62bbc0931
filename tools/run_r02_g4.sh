#!/bin/bash
# round 2, 4 GPUs: multi-GPU tests, bench self-launch (C2 strong, C3 weak), C4 on
# 4 GPUs with the packed store, and C4 on 2 of them
set -u
mkdir -p gpurun_out
free -g > gpurun_out/g4_topo.txt; nvidia-smi topo -m >> gpurun_out/g4_topo.txt 2>&1
python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs > gpurun_out/g4_tests.log 2>&1
echo "tests rc=$?"
python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g4_bench_c2.json 2> gpurun_out/g4_bench_c2.err
echo "bench c2 n4 rc=$?"
python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g2_bench_c2.json 2> gpurun_out/g2_bench_c2.err
echo "bench c2 n2 rc=$?"
python bench.py --gpus 4 --config c3 --steps 2 --warmup 3 --no-e2e > gpurun_out/g4_bench_c3.json 2> gpurun_out/g4_bench_c3.err
echo "bench c3 n4 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
    --master-port 29533 tools/c4_run.py > gpurun_out/g4_c4_right.json 2> gpurun_out/g4_c4_right.err
echo "c4 n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
    --master-addr 127.0.0.1 --master-port 29534 tools/c4_run.py > gpurun_out/g2_c4_right.json 2> gpurun_out/g2_c4_right.err
echo "c4 n2 rc=$?"
