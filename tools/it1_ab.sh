#!/bin/bash
# 1 GPU: C3 iteration 1 (the heaviest) split-path A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in "MCLX_DUMMY=1" "MCLX_SPLIT_PRIVATE=0" "MCLX_SPLIT_CAND=0"; do
  env $v python bench.py --iters 1 --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$v', round(d['value'],1), round(d['ms_per_step'],2), round(c['split']['ms'],1), c['split']['items'], [round(x,1) for x in c['split']['variant_ms']])"
done
