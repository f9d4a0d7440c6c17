# K3 work-unit size sweep on the config-4 deep step (diagnostics): groups of
# 32 words per persistent-warp unit; K3 time per launch from the live profile
for u in ${UNITS:-4 8 16}; do  # forced sizes; the default picks 4 (config 2) or 16 (config 4)
  make -s -C paper_2511_20975_b200/csrc EXTRA=-DAG_UNIT_GROUPS=$u -B > /dev/null 2>&1
  echo "unit $u: $(timeout 300 python bench.py --steps 5 --warmup 3 --no-sched --no-cpu-baseline --no-config5 --no-noisy --no-chain --no-linear --no-select --no-ubench | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["detail"]["deep"]["ms_per_step"], d["detail"]["deep"]["kernel_ms"]["k_route_compact"])')"
done
make -s -C paper_2511_20975_b200/csrc -B > /dev/null 2>&1
