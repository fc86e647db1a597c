#!/bin/bash
# development: GPU parity + bench, then kernel counters with the -DMCLX_PROF build
bash tools/gpu_check.sh
cp paper_2002_10083_b200/libmclx.so /tmp/lib_keep.so
cp tools/libmclx_prof.so paper_2002_10083_b200/libmclx.so && python tools/prof_counters.py C3 -1,3,4 2>&1 | grep force_bin
cp /tmp/lib_keep.so paper_2002_10083_b200/libmclx.so
