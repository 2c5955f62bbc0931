#!/bin/bash
# Round-1 re-measurement after the balanced multi-GPU W solve (gpurun --gpus 4).
set -u
mkdir -p gpurun_out
P=127.0.0.1
run() {  # run <n> <outfile> <args...>
  local n=$1 out=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py "$@" > gpurun_out/$out 2> gpurun_out/$out.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr $P \
      --master-port $((29600 + n)) bench.py --gpus $n "$@" > gpurun_out/$out 2> gpurun_out/$out.err
  fi
  echo "$out rc=$? $(tail -c 200 gpurun_out/$out)"
}
run 1 f2_c2_n1.json
run 2 f2_c2_n2.json
run 4 f2_c2_n4.json
run 2 f2_c3_n2.json --config c3
run 4 f2_c3_n4.json --config c3
