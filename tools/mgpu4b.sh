#!/bin/bash
# 4-GPU: parity of the pipelined staged SUMMA (2x2) and its bench line
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29512 tools/mgpu_check.py --grids 2x2 > gpurun_out/mg4b_check.log 2>&1; echo check rc=$?
grep -E "PASS|FAIL" gpurun_out/mg4b_check.log; tail -3 gpurun_out/mg4b_check.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29514 bench.py --gpus 4 --grid 2x2 --steps 5 --warmup 3 > gpurun_out/mg4b_2x2.json 2> gpurun_out/mg4b_2x2.err; echo bench 2x2 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/mg4b_2x2.json').read().strip().splitlines()[-1]); print('2x2', round(d['value'],1), round(d['ms_per_step'],1), d['config']['ms_raw'], d['e2e'])"
tail -2 gpurun_out/mg4b_2x2.err
