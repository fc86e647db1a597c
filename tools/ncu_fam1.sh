#!/bin/bash
# ncu --set full of the CTA-shared-table family's bin-4 kernel on the C3 step (MCLX_FAMILY=1)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export MCLX_FAMILY=1
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pre_fam1.json 2>&1; echo pre rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:[(]int[)]8192, [(]int[)]512, [(]int[)]2, [(]bool[)]0, [(]bool[)]1' -c 1 -o gpurun_out/fam1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_fam1.log 2>&1; echo ncu rc=$?
