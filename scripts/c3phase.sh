#!/bin/bash
# Phase-timer build of the scheduler (diagnostics): per-round setup / first
# chunk / walk / finalize and per-step find / lists / merge / adopt cycles.
# usage (under gpurun): bash scripts/c3phase.sh <tag> [beam ...]
# C3_EXTRA: more -D flags for the diagnostic build (e.g. -DAG_SCHED_WAITPROD=1)
tag=${1:-rXX}; shift
touch paper_2511_20975_b200/csrc/ag_sched.cu
make -s -C paper_2511_20975_b200/csrc EXTRA="-DAG_SCHED_PHASE_TIMERS=1 $C3_EXTRA" > /dev/null
for b in ${@:-4 1}; do
  C3_ROUNDS=60 python scripts/c3phase.py $b > gpurun_out/${tag}_c3phase_b$b.txt 2>&1
done
touch paper_2511_20975_b200/csrc/ag_sched.cu
make -s -C paper_2511_20975_b200/csrc > /dev/null
