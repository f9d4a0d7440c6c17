#!/bin/bash
# Round-2 ncu captures (one GPU; never multi-rank): scheduler round kernel
# (B = 4 and B = 1, round 6 = 64 free slots) with source-level warp sampling,
# the runtime-cost argmin kernels, k_predict, k_sched_prune, and the learned
# router with its tensor-pipe counters.  usage: bash scripts/ncu_r02.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N --warp-sampling-interval 0 -k regex:k_sched_round -s 6 -c 1 -o gpurun_out/${tag}_sched4 python scripts/sched_ncu.py 8 4 > /dev/null 2>&1
timeout 600 $N --warp-sampling-interval 0 -k regex:k_sched_round -s 6 -c 1 -o gpurun_out/${tag}_sched1 python scripts/sched_ncu.py 8 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_sched_prune -s 4 -c 2 -o gpurun_out/${tag}_prune python scripts/sched_ncu.py 8 4 > /dev/null 2>&1
timeout 600 $N -k regex:"k_cost|k_predict" -s 12 -c 5 -o gpurun_out/${tag}_cost python scripts/select_probe.py > /dev/null 2>&1
timeout 600 $N --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:k_linear_score -s 2 -c 1 -o gpurun_out/${tag}_linear python scripts/linear_probe.py > /dev/null 2>&1
ls -la gpurun_out | grep $tag
