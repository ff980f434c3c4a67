# A/B of engine builds (paper_2510_03996_b200/_lib/ab/<variant>.so): sparse bootstrap times
for v in ${AB_VARIANTS:-base u1 u2 u3 u4 u5 base}; do
  echo "== $v"
  FHEON_LIB_OVERRIDE=paper_2510_03996_b200/_lib/ab/$v.so timeout 300 python scripts/boot_sparse_time.py 2>&1 | grep "bootstrap active"
done
