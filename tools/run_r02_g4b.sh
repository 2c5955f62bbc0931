#!/bin/bash
# 4 GPUs, every command bounded: look-ahead debug (the bench engine sequence),
# the C2 bench at 4 and 2 GPUs (default schedule), C3 weak at 2, the
# multi-GPU suite
set -u
mkdir -p gpurun_out
DSEL_LOOKAHEAD=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
    --master-port 29571 tools/debug/la_bench_like.py full > gpurun_out/g4b_la_dbg.log 2>&1
echo "la debug rc=$?"
for r in 0 1 2 3; do tail -2 gpurun_out/la_dbg_r$r.log 2>/dev/null; done
timeout 600 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/g4b_bench_c2_n4.json 2> gpurun_out/g4b_bench_c2_n4.err
echo "bench c2 n4 rc=$?"
timeout 900 python bench.py --gpus 2 --config c3 --steps 2 --warmup 3 --no-e2e > gpurun_out/g4b_bench_c3_n2.json 2> gpurun_out/g4b_bench_c3_n2.err
echo "bench c3 n2 rc=$?"
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs > gpurun_out/g4b_tests.log 2>&1
echo "mg tests rc=$?"
tail -3 gpurun_out/g4b_tests.log
