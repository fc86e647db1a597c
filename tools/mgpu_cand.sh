#!/bin/bash
# 4 GPUs: candidate-mode (fused) accumulating 2D SUMMA -- parity on 2x2 / 4x1 / phased 2x2 /
# 2x1, then C3 / C5 / C4 iteration times at 2x2 (C4 also unfused for comparison)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2_cand
O=gpurun_out/r2_cand
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run_check() {
  local np=$1 grids=$2 tag=$3; shift 3
  env "$@" timeout 900 $TR --nproc-per-node $np --master-port $((29500 + RANDOM % 400)) \
      tools/mgpu_check.py --grids $grids > $O/mg_$tag.log 2>&1
  echo "check $tag rc=$?"; grep -E "PASS|FAIL" $O/mg_$tag.log
}
run_bench() {
  local np=$1 cfg=$2 grid=$3 tag=$4 steps=$5 warm=$6; shift 6
  env PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True "$@" timeout 1500 $TR --nproc-per-node $np \
      --master-port $((29500 + RANDOM % 400)) bench.py \
      --gpus $np --config $cfg --grid $grid --steps $steps --warmup $warm --e2e-steps 0 \
      > $O/mgb_$tag.json 2> $O/mgb_$tag.err
  echo "bench $tag rc=$?"
  python -c "import json; d=json.loads(open('$O/mgb_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['ms_per_step'],2), 'phases', d['config'].get('phases'))"
}
run_check 4 2x2,4x1 n4
run_check 4 2x2 n4_phases MCLX_PHASES=3 MCLX_SUMMA_STAGES=2
run_check 2 2x1 n2
run_bench 4 C3 2x2 c3_2x2 5 3
run_bench 4 C5 2x2 c5_2x2 3 2
run_bench 4 C3 4x1 c3_4x1 5 3
run_bench 4 C4 2x2 c4_2x2 1 1
