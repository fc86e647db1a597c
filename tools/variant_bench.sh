#!/bin/bash
# A/B kernel variants: swap prebuilt libmclx.so files and run the bench (development aid)
cp paper_2002_10083_b200/libmclx.so /tmp/lib_cur.so
for v in tools/variants/*.so; do
  cp $v paper_2002_10083_b200/libmclx.so
  python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value'],1), [round(x,1) for x in d['config']['bin_ms']])"
done
cp /tmp/lib_cur.so paper_2002_10083_b200/libmclx.so
