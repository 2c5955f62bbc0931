#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
    --master-port 29581 tests/mp_engine_check.py lookahead > gpurun_out/g2c_mp_la.log 2>&1
echo "mp lookahead rc=$?"; grep rank gpurun_out/g2c_mp_la.log
DSEL_LOOKAHEAD=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
    --master-port 29582 tools/debug/la_bench_like.py full > gpurun_out/g2c_la_dbg.log 2>&1
echo "la debug rc=$?"
for r in 0 1; do grep time_to_k gpurun_out/la_dbg_r$r.log; done
DSEL_LOOKAHEAD=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g2c_bench_la.json 2> gpurun_out/g2c_bench_la.err
echo "bench la rc=$?"
