#!/bin/bash
# Source-level ncu captures (one GPU): k_route_compact (config-2 routing),
# k_cost_tasks (config-4 argmin) and the B = 4 scheduler round (round 6,
# 64 free slots).  usage: bash scripts/ncu_r02b.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:k_route_compact -s 2 -c 1 -o gpurun_out/${tag}_compact python bench.py --no-sched --no-deep --no-cpu-baseline --no-config5 --no-ubench --no-noisy --no-chain --no-linear --no-select --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_cost_tasks -s 2 -c 1 -o gpurun_out/${tag}_costtasks python scripts/deep_probe.py > /dev/null 2>&1
timeout 600 $N --warp-sampling-interval 0 -k regex:k_sched_round -s 6 -c 1 -o gpurun_out/${tag}_sched4 python scripts/sched_ncu.py 8 4 > /dev/null 2>&1
ls -la gpurun_out | grep $tag
