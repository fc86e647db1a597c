#!/bin/bash
# 1 GPU: where do the occasional ~30 ms step outliers of the 1-GPU C3 bench come from?
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/stall
O=gpurun_out/stall
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],2), d['config']['step_ms'])"; }
for r in 1 2; do
  python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/def$r.json 2>/dev/null; show $O/def$r.json default$r
  PYTORCH_CUDA_ALLOC_CONF=expandable_segments:False python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/noexp$r.json 2>/dev/null; show $O/noexp$r.json noexp$r
done
