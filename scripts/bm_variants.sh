# bitmap argmin variants (diagnostics): words per warp task
for v in 4096 2048 512 256; do
  make -s -C paper_2511_20975_b200/csrc "EXTRA=-DAG_BM_TASK=$v" -B > /dev/null 2>&1
  echo "task $v"; timeout 300 python scripts/bm_probe.py 2>&1 | tail -4 | cut -c1-130
done
make -s -C paper_2511_20975_b200/csrc -B > /dev/null 2>&1
