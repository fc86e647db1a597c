#!/bin/bash
# 1 GPU: bin sizing A/B on C3 it0 -- MCLX_MAX_LOAD (bin when need <= load x cap) and MCLX_ALPHA
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in "0.5 1.2" "0.6 1.2" "0.7 1.2" "0.5 1.1" "0.6 1.1" "0.45 1.2"; do
  set -- $v
  MCLX_MAX_LOAD=$1 MCLX_ALPHA=$2 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('load $1 alpha $2', round(d['value'],1), round(d['ms_per_step'],2), [round(x,2) for x in c['bin_ms']], c['bin_cols'], 'retries', c['retries'])"
done
