# A/B of engine builds (paper_2510_03996_b200/_lib/ab/<variant>.so): sparse bootstrap + ResNet-20 times
for v in ${AB_VARIANTS:-base new base new}; do
  echo "== $v"
  FHEON_LIB_OVERRIDE=paper_2510_03996_b200/_lib/ab/$v.so timeout 300 python scripts/boot_sparse_time.py ${AB_ARGS} 2>&1 | grep -E "bootstrap active|resnet20 boot_sparse 3"
done
