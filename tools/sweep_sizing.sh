for cfg in "1.2 0.5" "1.0 0.5" "1.2 0.35" "1.2 0.7" "1.0 0.7" "1.5 0.25"; do
  set -- $cfg
  MCLX_ALPHA=$1 MCLX_MAX_LOAD=$2 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('alpha=$1 load=$2', round(d['value'],1), 'GF/s', [round(x,1) for x in d['config']['bin_ms']], 'retries', d['config']['retries'])"
done
