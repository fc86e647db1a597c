#!/bin/bash
# 4 GPUs: C4 (R-MAT scale 22) iteration 0 at 2x2 (candidate-mode SUMMA) and on 1 GPU
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2_final
O=gpurun_out/r2_final
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --config C4 --steps 1 --warmup 1 \
    --e2e-steps 0 --no-cpu-baseline > $O/c4_2x2.json 2> $O/c4_2x2.err
echo "2x2 rc=$?"; tail -1 $O/c4_2x2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 2x2', round(d['value'],1), round(d['ms_per_step'],1), d['config'].get('summa_ms'), d['config']['phases'])"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --config C4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/c4_n1.json 2> $O/c4_n1.err
echo "n1 rc=$?"; tail -1 $O/c4_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 1 GPU', round(d['value'],1), round(d['ms_per_step'],1))"
