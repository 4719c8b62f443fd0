#!/bin/bash
# Bench lines of the paper's own kernel designs and of the fused pipeline
# at class A on one GPU, next to the product line.
# Usage (under gpurun): bash tools/ablation_bench.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu "$@" > gpurun_out/abl_${TAG}_$name.log 2>&1; echo "$name rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/abl_${TAG}_$name.log | head -1)"; }
run product
run charge_mode1 --charge-mode 1
run charge_mode2 --charge-mode 2
run push_mode1 --push-mode 1
run fused --fused
