#!/bin/bash
# 4 GPUs: distributed-prune changes -- 1-GPU phase / SUMMA / hostmem tests, torchrun parity,
# C3 / C5 2x2 timing
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2_final
O=gpurun_out/r2_final
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_phases.py -q -x > $O/phases_tests.log 2>&1
echo "phases rc=$?"; tail -1 $O/phases_tests.log
bash tools/mgpu_quick.sh
