#!/bin/bash
# 1 GPU: epilogue / accumulate cycle split (MCLX_PROF build), per-iteration C3 full-MCL times
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
cp paper_2002_10083_b200/libmclx.so /tmp/lib_keep.so
cp tools/libmclx_prof.so paper_2002_10083_b200/libmclx.so
python tools/prof_counters.py C3 -1 > gpurun_out/prof_counters.log 2>&1; echo prof rc=$?
cp /tmp/lib_keep.so paper_2002_10083_b200/libmclx.so
python tools/mcl_times.py C3 > gpurun_out/mcl_times_C3.jsonl 2>&1; echo times rc=$?
tail -1 gpurun_out/prof_counters.log; tail -1 gpurun_out/mcl_times_C3.jsonl
