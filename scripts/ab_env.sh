# A/B of an environment switch: sparse bootstrap times with ${AB_ENV}=0 and =1
for v in 0 1 0 1; do
  echo "== ${AB_ENV}=$v"
  env ${AB_ENV}=$v timeout 300 python scripts/boot_sparse_time.py 2>&1 | grep "bootstrap active"
done
