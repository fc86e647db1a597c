#!/bin/bash
# one GPU call: parity tests then the bench (used during development)
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
