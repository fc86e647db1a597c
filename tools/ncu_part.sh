#!/bin/bash
# ncu --set full of the split-part kernel (CTA-shared family, kPart) at C3 iteration 1
python bench.py --iters 1 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pre_part.json 2>&1; echo pre rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:[(]int[)]8192, [(]int[)]512, [(]int[)]3' --launch-skip 10 -c 1 -o gpurun_out/part_it1 \
    python bench.py --iters 1 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_part.log 2>&1; echo ncu rc=$?
