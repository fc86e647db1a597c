#!/bin/bash
# A/B the prebuilt tools/variants/*.so on C3 it0 and C3 it1 (development aid)
mkdir -p gpurun_out
bash tools/variant_bench.sh > gpurun_out/var_it0.log 2>&1
cp paper_2002_10083_b200/libmclx.so /tmp/lib_cur.so
for v in tools/variants/*.so; do
  cp $v paper_2002_10083_b200/libmclx.so
  python bench.py --iters 1 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v it1', round(d['value'],1), [round(x,1) for x in d['config']['bin_ms']])" >> gpurun_out/var_it1.log
done
cp /tmp/lib_cur.so paper_2002_10083_b200/libmclx.so
cat gpurun_out/var_it0.log gpurun_out/var_it1.log
