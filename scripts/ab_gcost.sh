# planner giant-cost sweep: sparse bootstrap times and keys
for gc in ${GCOSTS:-6.7 8.5 12 8.5}; do
  echo "== gcost $gc"
  FHEON_DH_GCOST=$gc timeout 300 python scripts/boot_sparse_time.py 2>&1 | grep -E "bootstrap active|keys"
done
