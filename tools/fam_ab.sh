cd "$GRAFT_REPO_ROOT"
for f in -1 1; do MCLX_FAMILY=$f python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('family $f', round(d['value'],1), [round(x,2) for x in d['config']['bin_ms']])"; done
