#!/bin/bash
# 4 GPUs with the final gain kernel: the Nt = 420 multi-GPU goldens (c3, c3mini) + look-ahead + peer failure
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_cpp_dropin.py -m gpu -q -rs -k "c3 or lookahead or fault" > gpurun_out/g4h_tests.log 2>&1
echo "mg tests rc=$?"; tail -2 gpurun_out/g4h_tests.log
