#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --config C4 --grid 2x2 --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/mgc_c4_2x2.json 2> gpurun_out/mgc_c4_2x2.err
echo "c4 2x2 rc=$?"; tail -1 gpurun_out/mgc_c4_2x2.json | python -c "import json,sys; d=json.load(sys.stdin); print('c4_2x2', round(d['value'],1), round(d['ms_per_step'],1), 'phases', d['config'].get('phases'))"
grep -i "error" gpurun_out/mgc_c4_2x2.err | head -3
