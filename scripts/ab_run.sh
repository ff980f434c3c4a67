#!/bin/bash
# A/B the library variants under build_ab/ against the in-tree build:
# NTT microbench (+ bit-exact primitives, + ResNet-20 with AB_RESNET=1) for each.
for v in base $(ls build_ab 2>/dev/null); do
  if [ "$v" = base ]; then unset FHEON_LIB_OVERRIDE; else export FHEON_LIB_OVERRIDE=$PWD/build_ab/$v/libfheon_b200.so; fi
  echo "== $v"
  timeout 120 python scripts/ntt_time.py 2>&1 | tail -2
  if [ -n "$AB_TESTS" ]; then timeout 300 python -m pytest tests/test_gpu_primitives.py -q -x 2>&1 | tail -1; fi
  if [ -n "$AB_RESNET" ]; then timeout 300 python scripts/warm_probe.py 12 4 2>&1 | grep -v slowest | tail -1 | cut -c1-40; fi
done
