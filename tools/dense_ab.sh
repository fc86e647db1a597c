#!/bin/bash
# dense-sweep threshold A/B on C4 at scale 20 (and 22 with DENSE_AB_22=1)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for p in 64 32 16 8; do
  MCLX_DENSE_MIN_P=$p python tools/c4s20_once.py 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('minP $p', round(sum(d['bin_ms'])/1e3,3), 's', d['split_vcols'], [round(x/1e3,3) for x in d['split_vms']])"
done
