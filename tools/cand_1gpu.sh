#!/bin/bash
# 1 GPU: candidate-mode (fused) accumulating SUMMA on a forced 1 x 1 grid -- parity tests,
# then C3 iteration time of the accumulating form fused vs unfused vs the 1-GPU iteration
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phases.py -x -q > gpurun_out/cand_phases.log 2>&1
echo "phases rc=$?"; tail -3 gpurun_out/cand_phases.log
for v in fused unfused; do
  if [ $v = unfused ]; then X="MCLX_SUMMA_UNFUSED=1"; else X="MCLX_DUMMY=1"; fi
  env MCLX_SUMMA_ACCUM=1 $X timeout 600 python tools/summa1x1_time.py C3 5 > gpurun_out/cand_c3_$v.log 2>&1
  echo "c3 $v rc=$?"; tail -3 gpurun_out/cand_c3_$v.log
done
