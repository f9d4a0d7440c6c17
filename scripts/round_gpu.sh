#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), ncu launch list and full
# captures of the dominant kernels (routing, scheduler round, learned router,
# noisy router, argmin, predict, prune).
# usage (under gpurun): bash scripts/round_gpu.sh <tag>
tag=${1:-rXX}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
Q="--no-sched --no-deep --no-cpu-baseline --no-config5 --no-ubench --no-select"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 3 $Q --no-noisy --no-chain --no-linear > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:k_route -s 8 -c 4 -o gpurun_out/${tag}_route python bench.py $Q --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_sched_round -s 6 -c 1 -o gpurun_out/${tag}_sched python scripts/sched_ncu.py 8 > /dev/null 2>&1
timeout 600 $N --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active -k regex:k_linear_score -s 2 -c 1 -o gpurun_out/${tag}_linear python scripts/linear_probe.py > /dev/null 2>&1
timeout 600 $N -k regex:k_route_noise -s 1 -c 1 -o gpurun_out/${tag}_noise python scripts/noisy_ncu.py > /dev/null 2>&1
timeout 600 $N -k regex:"k_cost|k_predict" -s 12 -c 6 -o gpurun_out/${tag}_cost python scripts/select_probe.py > /dev/null 2>&1
timeout 600 $N -k regex:k_sched_prune -s 4 -c 2 -o gpurun_out/${tag}_prune python scripts/sched_ncu.py 8 4 > /dev/null 2>&1
./scripts/ubench/bw > gpurun_out/${tag}_ubench.txt 2>&1
./scripts/ubench/mix_peak >> gpurun_out/${tag}_ubench.txt 2>&1
ls -la gpurun_out | grep ${tag} | tail -30
