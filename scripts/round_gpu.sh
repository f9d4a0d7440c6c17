#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), ncu launch list and full
# captures of the dominant routing kernels and the scheduler round kernel.
# usage (under gpurun): bash scripts/round_gpu.sh <tag>
tag=${1:-rXX}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-sched --no-deep --no-cpu-baseline --no-config5 --no-noisy --no-chain --no-linear --no-ubench > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_route -s 8 -c 4 -o gpurun_out/${tag}_route \
  python bench.py --no-sched --no-deep --no-cpu-baseline --no-config5 --no-ubench --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sched_round -s 6 -c 1 -o gpurun_out/${tag}_sched \
  python scripts/sched_ncu.py 8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_linear_score -s 2 -c 1 -o gpurun_out/${tag}_linear \
  python scripts/linear_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_route_noise -s 1 -c 1 -o gpurun_out/${tag}_noise \
  python scripts/noisy_ncu.py > /dev/null 2>&1
./scripts/ubench/bw > gpurun_out/${tag}_ubench.txt 2>&1
./scripts/ubench/mix_peak >> gpurun_out/${tag}_ubench.txt 2>&1
ls -la gpurun_out | tail -20
