# A/B of engine builds in one box session: paper_2510_03996_b200/_lib/ab/<variant>.so
for v in ${AB_VARIANTS:-base new base new}; do FHEON_LIB_OVERRIDE=paper_2510_03996_b200/_lib/ab/$v.so timeout 300 python scripts/ab_time.py $v ${AB_WHAT:-all} 2>&1 | tail -1; done
