for v in "" nopre; do
  echo "== variant ${v:-prod}"
  for m in 0 1 2; do
    QOQ_LIB_VARIANT=$v QOQ_FORCE_MODE=$m timeout 60 python tools/prof_gemm.py --M 64 --N 4096 --K 4096 --time 2>&1 | tail -1 | cut -c1-150
  done
done
