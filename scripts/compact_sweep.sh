# K3 work-unit size sweep (diagnostics): groups of 32 words per persistent-warp unit
for u in ${UNITS:-2 4 8 16 32}; do
  make -s -C paper_2511_20975_b200/csrc EXTRA=-DAG_UNIT_GROUPS=$u -B > /dev/null 2>&1
  echo "unit $u: $(timeout 120 python bench.py --steps 10 --warmup 3 --no-sched --no-deep --no-cpu-baseline --no-config5 --no-noisy --no-chain --no-linear --no-select --no-ubench | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["avg_launch_ms"])')"
done
make -s -C paper_2511_20975_b200/csrc -B > /dev/null 2>&1
