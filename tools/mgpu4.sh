#!/bin/bash
# 4-GPU checks: SUMMA parity (1x4, 2x2) and N=4 bench lines (C3, C5)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29512 tools/mgpu_check.py --grids 1x4,2x2 > gpurun_out/mg4_check.log 2>&1; echo check rc=$?
grep -E "PASS|FAIL" gpurun_out/mg4_check.log
for cfg in C3 C5; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 4 --config $cfg --steps 5 --warmup 3 > gpurun_out/mg4_$cfg.json 2> gpurun_out/mg4_$cfg.err; echo bench $cfg rc=$?
python -c "import json; d=json.loads(open('gpurun_out/mg4_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value'],1), round(d['ms_per_step'],1), d['e2e'])"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29514 bench.py --gpus 4 --grid 2x2 --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/mg4_2x2.json 2> gpurun_out/mg4_2x2.err; echo bench 2x2 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/mg4_2x2.json').read().strip().splitlines()[-1]); print('2x2', round(d['value'],1), round(d['ms_per_step'],1))"
