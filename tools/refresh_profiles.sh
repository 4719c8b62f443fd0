#!/bin/bash
# Round-end measurement set (run under gpurun, 1 GPU): the bench line, the ncu
# launch list of the same command, and one ncu --set full capture of the two
# dominant kernels (deposit + push, both stages).  Each ncu pass runs only
# after its command exited 0 without ncu.  Usage: tools/refresh_profiles.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; rc=$?
echo "bench rc=$rc"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
timeout 300 python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_short_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/prof_step.py --size A --steps 1 --warmup 1 > gpurun_out/prof_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_deposit_tiled|k_push" -s 1 -c 4 \
    -o gpurun_out/kernels_$TAG python tools/prof_step.py --size A --steps 1 --warmup 1 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
