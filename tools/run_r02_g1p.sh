#!/bin/bash
# reciprocal pivot chain in the diagonal-block factorization: GPU parity + gain-phase times (C2, C3)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_storage_edges.py tests/test_gpu_parity.py tests/test_cli.py -m gpu -q -x -rs > gpurun_out/g1p_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/g1p_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1p_smoke.log 2>&1; echo "smoke rc=$?"
DSEL_LOOKAHEAD=0 timeout 300 python tools/profile_c2.py --runs 2 > gpurun_out/g1p_c2.json 2>&1
echo "c2 rc=$? $(python -c "import json;j=json.load(open('gpurun_out/g1p_c2.json'));print(j['time_to_k_ms'],j['phase_ms']['ms_gain'])")"
timeout 300 python tools/profile_c2.py --nd 75 --nt 420 --rank 24576 --runs 2 > gpurun_out/g1p_c3.json 2>&1
echo "c3 rc=$? $(python -c "import json;j=json.load(open('gpurun_out/g1p_c3.json'));print(j['time_to_k_ms'],j['phase_ms']['ms_gain'])")"
