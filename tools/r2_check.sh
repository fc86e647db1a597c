#!/bin/bash
# round-2 quick check on the GPU box: error-path tests, a parity subset, bench line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests/test_gpu_errors.py tests/test_gpu_parity.py -x -q -m gpu -k "not slow" > gpurun_out/r2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_tests.log
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?"
