#!/bin/bash
# round 2, 2 GPUs: multi-GPU tests (G-invariance, peer-failure abort), the bench
# self-launch at --gpus 2, C3 weak at 2, and C4 (600 x 420, select 175) on 2 GPUs
# with the packed block-lower store (127 GB of panels per GPU)
set -u
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/g2_topo.txt 2>&1; free -g >> gpurun_out/g2_topo.txt
python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs > gpurun_out/g2_tests.log 2>&1
echo "tests rc=$?"
python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g2_bench_c2.json 2> gpurun_out/g2_bench_c2.err
echo "bench c2 rc=$?"
python bench.py --gpus 2 --config c3 --steps 2 --warmup 3 --no-e2e > gpurun_out/g2_bench_c3.json 2> gpurun_out/g2_bench_c3.err
echo "bench c3 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
    --master-port 29533 tools/c4_run.py > gpurun_out/g2_c4_right.json 2> gpurun_out/g2_c4_right.err
echo "c4 rc=$?"
