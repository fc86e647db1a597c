#!/bin/bash
# A/B variants on C3 it1 and C4 scale 20 (development aid)
cp paper_2002_10083_b200/libmclx.so /tmp/lib_cur.so
for v in tools/variants/*.so; do
  cp $v paper_2002_10083_b200/libmclx.so
  python bench.py --iters 1 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v it1', round(d['value'],1), d['config']['split']['variant_ms'])"
  python bench.py --config C4 --scale 0.25 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v c4s20', round(d['value'],1), d['config']['split']['variant_ms'])"
done
cp /tmp/lib_cur.so paper_2002_10083_b200/libmclx.so
