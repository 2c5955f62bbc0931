#!/bin/bash
# look-ahead validation and timing: 1-GPU parity, C2 with / without, then the
# multi-GPU check and the C2 bench at every GPU count the box has
set -u
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python -m pytest tests/test_gpu_storage_edges.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/la_tests.log 2>&1
echo "tests rc=$?"
DSEL_LOOKAHEAD=0 python tools/profile_c2.py --runs 2 > gpurun_out/la_off.json 2>&1
python tools/profile_c2.py --runs 2 > gpurun_out/la_on.json 2>&1
for r in 8 24; do DSEL_LA_RESERVE=$r python tools/profile_c2.py --runs 2 > gpurun_out/la_on_r$r.json 2>&1; done
if [ "$N" -ge 2 ]; then
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29561 \
      tests/mp_engine_check.py lookahead > gpurun_out/la_mp.log 2>&1
  echo "mp lookahead rc=$?"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29562 \
      tests/mp_engine_check.py c2 > gpurun_out/la_mp_c2.log 2>&1
  echo "mp c2 rc=$?"
  for g in 2 $N; do
    python bench.py --gpus $g --steps 3 --warmup 3 --no-cpu --no-variants > gpurun_out/la_bench_n$g.json 2> gpurun_out/la_bench_n$g.err
    DSEL_LOOKAHEAD=0 python bench.py --gpus $g --steps 3 --warmup 3 --no-cpu --no-variants --no-e2e > gpurun_out/la_off_bench_n$g.json 2> gpurun_out/la_off_bench_n$g.err
  done
fi
echo done
