#!/bin/bash
# final 1-GPU check of the committed code: full GPU suite + smoke
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/g1t_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/g1t_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1t_smoke.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/g1t_smoke.log
