#!/bin/bash
# ncu --set full of one dense-row-tile launch (k_dense_part<float>) at C4 scale 20
python bench.py --config C4 --scale 0.25 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pre_dense.json 2>&1; echo pre rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_dense_part' --launch-skip 3 -c 1 -o gpurun_out/dense_c4 \
    python bench.py --config C4 --scale 0.25 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_dense.log 2>&1; echo ncu rc=$?
