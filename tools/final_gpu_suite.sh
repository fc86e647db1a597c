#!/bin/bash
# 1 GPU: the driver's round-end GPU tiers -- pytest -m gpu (with durations), smoke(), bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > $O/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -32 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?"; tail -c 1500 $O/bench.json
