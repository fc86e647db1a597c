#!/bin/bash
# 4 GPUs: C5 / C3 accumulating 2x2 with the 48 GB slot budget, and C4 (R-MAT scale 22)
# iteration times at 1x4 (fused) and 2x2 (accumulating, phased)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run_bench() {
  local np=$1 cfg=$2 grid=$3 tag=$4 steps=$5 warm=$6; shift 6
  env "$@" timeout 1500 $TR --nproc-per-node $np --master-port $((29500 + RANDOM % 400)) bench.py \
      --gpus $np --config $cfg --grid $grid --steps $steps --warmup $warm --e2e-steps 0 \
      > gpurun_out/mgc_$tag.json 2> gpurun_out/mgc_$tag.err
  echo "bench $tag rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/mgc_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'phases', d['config'].get('phases'))"
}
run_bench 4 C5 2x2 c5_2x2 3 2
run_bench 4 C3 2x2 c3_2x2 5 3
run_bench 4 C4 1x4 c4_1x4 1 1
run_bench 2 C4 1x2 c4_1x2 1 1
run_bench 4 C4 2x2 c4_2x2 1 1
