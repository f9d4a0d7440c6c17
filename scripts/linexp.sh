for e in ${EXPS:-0 1 2 3}; do
  make -s -C paper_2511_20975_b200/csrc EXTRA=-DAG_LIN_EXP=$e -B > /dev/null 2>&1
  echo "exp $e: $(timeout 120 python scripts/linear_probe.py)"
done
