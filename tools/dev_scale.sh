#!/bin/bash
# development: per-bin throughput with A resident in L2 (scale 0.25) vs full C3
for sc in 0.25 1.0; do
  MCLX_ORDER=0 python bench.py --scale $sc --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); c=d['config']
print('scale=$sc', round(d['value'],1), 'GF/s per bin', [round(f/1e6/max(m,1e-3),1) for f,m in zip(c['bin_flops'],c['bin_ms'])], 'ms', [round(x,1) for x in c['bin_ms']])"
done
