#!/bin/bash
# ESC on / off on a late C3 iteration (cf near 1) and on C3 it0
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for it in 0 8 14; do for cf in 0 1.5; do
MCLX_ESC_CF=$cf python bench.py --iters $it --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); c=d['config']
print('it$it cf$cf', round(d['value'],1), round(d['ms_per_step'],3), 'flops', c['flops_per_step'], [round(x,2) for x in c['bin_ms']], c.get('esc'))"
done; done
