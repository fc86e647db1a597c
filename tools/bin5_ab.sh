#!/bin/bash
# 1 GPU: route bin-5 columns (need 4096..8192) through the split path instead (A/B)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in default 4096 6144; do
  if [ $v = default ]; then X="MCLX_DUMMY=1"; else X="MCLX_SPLIT_MIN_NEED=$v"; fi
  env $X python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('$v', round(d['value'],1), round(d['ms_per_step'],2), [round(x,2) for x in c['bin_ms']], c['bin_cols'], round(c['split']['ms'],2), c['split']['items'], c['split']['variant_ms'])"
done
