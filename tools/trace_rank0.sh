#!/bin/bash
# torchrun --no-python target: host-gap tracing (MCLX_TRACE_SYNC) on local rank 0 only
if [ "$LOCAL_RANK" = "0" ]; then export MCLX_TRACE_SYNC=${TRACE_MS:-0.3}; fi
exec python bench.py "$@"
