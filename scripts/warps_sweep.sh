for w in 4 8 4 8; do
  make -s -C paper_2511_20975_b200/csrc EXTRA=-DAG_ROUTE_WARPS=$w -B > /dev/null 2>&1
  echo "warps $w: $(timeout 200 python bench.py --steps 10 --warmup 3 --no-sched --no-deep --no-cpu-baseline --no-config5 --no-chain --no-linear --no-ubench | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["kernel_share"], d["noisy"]["ms_per_step"], d["noisy"]["kernel_ms"])')"
done
