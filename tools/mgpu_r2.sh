#!/bin/bash
# round 2, 4 GPUs: SUMMA parity (2x2, 1x4, 4x1; 1x2 / 2x1 on 2 ranks; staged + phased
# variants) and the C3 / C5 bench lines at 2x2 (staged: Alg. 2 + distributed prune) and 1x4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run_check() {  # nproc grids tag [env...]
  local np=$1 grids=$2 tag=$3; shift 3
  env "$@" timeout 900 $TR --nproc-per-node $np --master-port $((29500 + RANDOM % 400)) \
      tools/mgpu_check.py --grids $grids > gpurun_out/mg_$tag.log 2>&1
  echo "check $tag rc=$?"; grep -E "PASS|FAIL" gpurun_out/mg_$tag.log
}
run_check 4 2x2,1x4,4x1 n4
run_check 4 2x2 n4_phases MCLX_PHASES=3 MCLX_SUMMA_STAGES=2
run_check 4 1x4 n4_staged MCLX_SUMMA_STAGED=1
run_check 2 1x2,2x1 n2
run_bench() {  # nproc cfg grid tag [env...]
  local np=$1 cfg=$2 grid=$3 tag=$4; shift 4
  env "$@" timeout 1200 $TR --nproc-per-node $np --master-port $((29500 + RANDOM % 400)) bench.py \
      --gpus $np --config $cfg --grid $grid --steps 5 --warmup 3 --e2e-steps 0 \
      > gpurun_out/mgb_$tag.json 2> gpurun_out/mgb_$tag.err
  echo "bench $tag rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/mgb_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('stage_ms'))"
}
run_bench 4 C3 2x2 c3_2x2
run_bench 4 C3 1x4 c3_1x4
run_bench 4 C5 2x2 c5_2x2
run_bench 4 C5 1x4 c5_1x4
run_bench 2 C3 1x2 c3_1x2
run_bench 2 C3 2x1 c3_2x1
