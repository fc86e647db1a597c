bash tools/variant_bench.sh
bash tools/dev_check.sh
