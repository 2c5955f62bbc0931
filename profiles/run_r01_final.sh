#!/bin/bash
# Round-1 closing check on one GPU (gpurun): GPU tests, smoke(), the default
# bench line and the reference arm, exactly as the driver runs them.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/fin_tests.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
echo "smoke rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
echo "ref rc=$? $(tail -c 200 gpurun_out/fin_ref.json)"
timeout 600 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
echo "bench rc=$? $(tail -c 200 gpurun_out/fin_bench.json)"
