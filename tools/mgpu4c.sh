#!/bin/bash
# 4-GPU: parity (1x4, 1x2 on 2 of the ranks' grid) and the C3 / C5 N=4 and N=2 bench lines
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29512 tools/mgpu_check.py --grids 1x4 > gpurun_out/mg4c_check.log 2>&1; echo check rc=$?
grep -E "PASS|FAIL" gpurun_out/mg4c_check.log
for cfg in C3 C5; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 4 --config $cfg --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/mg4c_$cfg.json 2> gpurun_out/mg4c_$cfg.err; echo bench $cfg rc=$?
python -c "import json; d=json.loads(open('gpurun_out/mg4c_$cfg.json').read().strip().splitlines()[-1]); print('$cfg N=4', round(d['value'],1), round(d['ms_per_step'],1), d['e2e'])"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29515 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/mg4c_n2.json 2> gpurun_out/mg4c_n2.err; echo bench n2 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/mg4c_n2.json').read().strip().splitlines()[-1]); print('C3 N=2', round(d['value'],1), round(d['ms_per_step'],1), d['e2e'])"
