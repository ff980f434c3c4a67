#!/bin/bash
# A/B the library variants under build_ab/ against the in-tree build:
# NTT microbench + ResNet-20 s/image for each.
for v in base $(ls build_ab 2>/dev/null); do
  if [ "$v" = base ]; then unset FHEON_LIB_OVERRIDE; else export FHEON_LIB_OVERRIDE=$PWD/build_ab/$v/libfheon_b200.so; fi
  echo "== $v"
  timeout 120 python scripts/ntt_time.py 2>&1 | tail -2
  if [ -n "$AB_RESNET" ]; then timeout 300 python scripts/resnet_breakdown.py resnet20 2>&1 | head -1; fi
done
