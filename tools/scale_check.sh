#!/bin/bash
# 4 GPUs: the driver's scaling commands with bench.py's defaults (north-star grids: 1x2 at
# N=2, 2x2 at N=4; e2e included), then N=4 at 1x4 for comparison
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2_scale
O=gpurun_out/r2_scale
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 10 --warmup 3 > $O/n1.json 2> $O/n1.err
echo "N=1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/n1_c5.json 2> $O/n1_c5.err
echo "N=1 C5 rc=$?"; tail -1 $O/n1_c5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 1 GPU', round(d['value'],1), round(d['ms_per_step'],2), round(d['config']['step_ms_max'],2))"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 400)) bench.py --gpus $N --steps 10 --warmup 3 > $O/n$N.json 2> $O/n$N.err
  echo "N=$N rc=$?"; tail -c 300 $O/n$N.json; echo
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --grid 1x4 --steps 10 --warmup 3 > $O/n4_1x4.json 2> $O/n4_1x4.err
echo "N=4 1x4 rc=$?"
python - <<'PY'
import json
for t in ["n1", "n2", "n4", "n4_1x4"]:
    try:
        d = json.loads(open(f"gpurun_out/r2_scale/{t}.json").read().strip().splitlines()[-1])
        print(t, d["config"]["parallelism"][:40], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 2),
              "e2e", d.get("e2e", {}).get("value"), "clocks", d.get("clocks", {}).get("sm_mhz"), "max step", round(d["config"]["step_ms_max"], 2),
              d["config"].get("summa_ms"))
    except Exception as e:
        print(t, "ERR", e)
PY
