#!/bin/bash
set -u
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
DSEL_LOOKAHEAD=1 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
    --master-port 29571 tools/debug/la_bench_like.py full > gpurun_out/la_dbg.log 2>&1
echo "la debug rc=$?"
for r in 0 1 2 3; do tail -3 gpurun_out/la_dbg_r$r.log 2>/dev/null; done
