#!/bin/bash
# 4 GPUs: accumulating 2D SUMMA (pr > 1 default) parity + bench, staged Alg. 2 for comparison
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run_check() {
  local np=$1 grids=$2 tag=$3; shift 3
  env "$@" timeout 900 $TR --nproc-per-node $np --master-port $((29500 + RANDOM % 400)) \
      tools/mgpu_check.py --grids $grids > gpurun_out/mg_$tag.log 2>&1
  echo "check $tag rc=$?"; grep -E "PASS|FAIL" gpurun_out/mg_$tag.log
}
run_bench() {
  local np=$1 cfg=$2 grid=$3 tag=$4; shift 4
  env "$@" timeout 1200 $TR --nproc-per-node $np --master-port $((29500 + RANDOM % 400)) bench.py \
      --gpus $np --config $cfg --grid $grid --steps 5 --warmup 3 --e2e-steps 0 \
      > gpurun_out/mgb_$tag.json 2> gpurun_out/mgb_$tag.err
  echo "bench $tag rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/mgb_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('stage_ms'), d['config'].get('phases'))"
}
run_check 4 2x2,4x1 acc_n4
run_check 4 2x2 acc_n4_phases MCLX_PHASES=3 MCLX_SUMMA_STAGES=2
run_check 2 2x1 acc_n2
run_bench 4 C3 2x2 acc_c3_2x2
run_bench 4 C5 2x2 acc_c5_2x2
run_bench 2 C3 2x1 acc_c3_2x1
run_bench 4 C3 4x1 acc_c3_4x1
python bench.py --config C5 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_c5.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b1_c5.json').read().strip().splitlines()[-1]); print('C5 1 GPU', round(d['value'],1), round(d['ms_per_step'],2))"
python bench.py --config C3 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_c3.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b1_c3.json').read().strip().splitlines()[-1]); print('C3 1 GPU', round(d['value'],1), round(d['ms_per_step'],2))"
