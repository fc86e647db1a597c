#!/bin/bash
# ncu --set full of the dominant launch (k_bin<8192,256,fused>) of the C3 bench step;
# optional $1 = a variant libmclx.so to profile instead of the built one
if [ -n "$1" ]; then cp paper_2002_10083_b200/libmclx.so /tmp/lib_keep.so; cp "$1" paper_2002_10083_b200/libmclx.so; fi
tag=${2:-b4}
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pre_$tag.json 2>&1; echo pre rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:[(]int[)]8192, [(]int[)]256, [(]int[)]2, [(]bool[)]0, [(]bool[)]0' -c 1 -o gpurun_out/$tag python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_$tag.log 2>&1; echo ncu rc=$?
if [ -n "$1" ]; then cp /tmp/lib_keep.so paper_2002_10083_b200/libmclx.so; fi
