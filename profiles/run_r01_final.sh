#!/bin/bash
# Round-1 final measurements (run under gpurun --gpus 4 on one B200 box).
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
run 1 bench_c2_n1.json
run 2 bench_c2_n2.json
run 4 bench_c2_n4.json
run 1 bench_c3_n1.json --config c3 --no-cpu
run 2 bench_c3_n2.json --config c3
run 4 bench_c3_n4.json --config c3
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
echo "ref rc=$? $(tail -c 300 gpurun_out/bench_ref_c2.json)"
for a in right left; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr $P \
    --master-port 29650 tools/c4_run.py --algorithm $a > gpurun_out/c4_g4_$a.log 2>&1
  echo "c4 $a rc=$? $(tail -c 300 gpurun_out/c4_g4_$a.log)"
done
