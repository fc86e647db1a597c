#!/bin/bash
# 2-GPU checks: SUMMA parity (grids 1x2, 2x1) and the N=2 bench line
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29512 tools/mgpu_check.py --grids 1x2,2x1 > gpurun_out/mg2_check.log 2>&1; echo check rc=$?
grep -E "PASS|FAIL" gpurun_out/mg2_check.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/mg2_bench.json 2> gpurun_out/mg2_bench.err; echo bench rc=$?
tail -c 600 gpurun_out/mg2_bench.json
