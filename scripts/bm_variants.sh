# bitmap argmin variants (diagnostics): words per lane per step x min blocks per SM
for v in "8 3" "16 2" "16 3" "4 4"; do
  set -- $v
  make -s -C paper_2511_20975_b200/csrc "EXTRA=-DAG_BM_RUN=$1 -DAG_BM_MINB=$2" -B > /dev/null 2>&1
  echo "run $1 minb $2"; timeout 300 python scripts/bm_probe.py 2>&1 | tail -4 | cut -c1-200
done
make -s -C paper_2511_20975_b200/csrc -B > /dev/null 2>&1
