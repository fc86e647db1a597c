#!/bin/bash
# development: A/B of the locality-ordered work lists
for o in 0 1; do
  MCLX_ORDER=$o python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('order=$o', round(d['value'],1), [round(x,1) for x in d['config']['bin_ms']], d['config']['stage_ms'])"
done
MCLX_ORDER=1 python tools/locality_probe.py
