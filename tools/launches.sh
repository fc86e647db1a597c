#!/bin/bash
# launch list (per-kernel device time) of a command: tools/launches.sh OUT.csv cmd...
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
out=$1; shift
"$@" > gpurun_out/launches_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out" "$@" > gpurun_out/launches_ncu.log 2>&1
echo rc=$?
