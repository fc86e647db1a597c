#!/bin/bash
# development: build libmclx.so and the -DMCLX_PROF copy (tools/libmclx_prof.so)
set -e
cd "$(dirname "$0")/.."
MCLX_NVCC_EXTRA=-DMCLX_PROF python paper_2002_10083_b200/_build.py
cp paper_2002_10083_b200/libmclx.so tools/libmclx_prof.so
python paper_2002_10083_b200/_build.py
