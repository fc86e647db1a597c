#!/bin/bash
# 1 GPU: MCLX_SPLIT_BIG (half the split parts, 16384-slot tables) A/B on C3 it1 / it0 + parity
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in 0 1; do
  for it in 1 0; do
    MCLX_SPLIT_BIG=$v python bench.py --iters $it --steps 5 --warmup 2 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('big=$v it$it', round(d['value'],1), round(d['ms_per_step'],2), round(c['split']['ms'],1), c['split']['items'], [round(x,1) for x in c['split']['variant_ms']])"
  done
done
MCLX_SPLIT_BIG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split or rmat or step_parity" 2>&1 | tail -2
