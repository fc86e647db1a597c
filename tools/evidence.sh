#!/bin/bash
# one GPU call that refreshes the round's evidence (bench lines, launch list, ncu capture)
mkdir -p gpurun_out
python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev_ncu_list.log 2>&1; echo list rc=$?
bash tools/ncu_bin4.sh "" ev_bin4 > /dev/null 2>&1; echo full rc=$?
python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev_c5.json 2> gpurun_out/ev_c5.err; echo c5 rc=$?
python bench.py --config C4 --scale 0.25 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev_c4s20.json 2> gpurun_out/ev_c4s20.err; echo c4 rc=$?
python bench.py --iters 1 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ev_c3it1.json 2> gpurun_out/ev_c3it1.err; echo c3it1 rc=$?
