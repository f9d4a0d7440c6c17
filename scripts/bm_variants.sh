# bitmap argmin variants (diagnostics): min blocks per SM
for v in 3 2; do
  make -s -C paper_2511_20975_b200/csrc "EXTRA=-DAG_BM_MINB=$v" -B > /dev/null 2>&1
  echo "minb $v"; timeout 300 python scripts/bm_probe.py 2>&1 | tail -4 | cut -c1-200
done
make -s -C paper_2511_20975_b200/csrc -B > /dev/null 2>&1
