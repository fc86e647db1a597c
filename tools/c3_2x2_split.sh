#!/bin/bash
# 4 GPUs: C3 2x2 step with the SUMMA time split (set-up / products / distributed prune)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2_scale
O=gpurun_out/r2_scale
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 10 --warmup 3 --e2e-steps 0 --config ${1:-C3} > $O/split_${1:-C3}.json 2> $O/split_${1:-C3}.err
echo "rc=$?"
tail -1 $O/split_${1:-C3}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print(d['ms_per_step'], c.get('summa_ms'), c['ms_raw'], sum(c['bin_ms']))"
