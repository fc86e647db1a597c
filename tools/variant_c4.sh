#!/bin/bash
# A/B the prebuilt tools/variants/*.so on C4 at R-MAT scale 20 (the CTA-shared family's workload)
mkdir -p gpurun_out
cp paper_2002_10083_b200/libmclx.so /tmp/lib_cur.so
for v in tools/variants/*.so; do
  cp $v paper_2002_10083_b200/libmclx.so
  python bench.py --config C4 --scale 0.25 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); c=d['config']; print('$v c4s20', round(d['value'],2), [round(x,1) for x in c['bin_ms']], c.get('split',{}).get('variant_ms'))" >> gpurun_out/var_c4.log
done
cp /tmp/lib_cur.so paper_2002_10083_b200/libmclx.so
cat gpurun_out/var_c4.log
