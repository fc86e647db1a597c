#!/bin/bash
# 4 GPUs: parity of the pr > 1 SUMMA (2x2, 4x1, phased 2x2) + C3 2x2 / C5 2x2 bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2_final
O=gpurun_out/r2_final
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) tools/mgpu_check.py --grids 2x2,4x1 > $O/mg_n4.log 2>&1
echo "check rc=$?"; grep -cE "PASS" $O/mg_n4.log; grep FAIL $O/mg_n4.log
MCLX_PHASES=3 MCLX_SUMMA_STAGES=2 timeout 900 $TR --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) tools/mgpu_check.py --grids 2x2 > $O/mg_n4_phases.log 2>&1
echo "check phases rc=$?"; grep -cE "PASS" $O/mg_n4_phases.log; grep FAIL $O/mg_n4_phases.log
for cfg in C3 C5; do
  timeout 900 $TR --nproc-per-node 4 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --config $cfg > $O/b4_$cfg.json 2> $O/b4_$cfg.err
  tail -1 $O/b4_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('summa_ms'))"
done
