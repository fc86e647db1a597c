#!/bin/bash
# A/B prebuilt tools/variants/*.so on C3 it0 (and it1 with AB_IT1=1), then optional tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
cp paper_2002_10083_b200/libmclx.so /tmp/lib_cur.so
for v in tools/variants/*.so; do
  cp $v paper_2002_10083_b200/libmclx.so
  for it in 0 ${AB_IT1:+1}; do
    timeout 600 python bench.py --iters $it --steps ${AB_STEPS:-5} --warmup 2 --no-cpu-baseline --e2e-steps 0 ${AB_ARGS} 2>>gpurun_out/ab_err.log | python -c "import json,sys; d=json.load(sys.stdin); print('$v it$it', round(d['value'],1), round(d['roofline']['frac'],3), [round(x,2) for x in d['config']['bin_ms']], d['config']['split']['ms'])" >> gpurun_out/ab.log
  done
done
cp /tmp/lib_cur.so paper_2002_10083_b200/libmclx.so
cat gpurun_out/ab.log
if [ -n "$AB_K" ]; then timeout 1200 python -m pytest tests -x -q -m gpu -k "$AB_K" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log; fi
