#!/bin/bash
# tensor-core basis conversion: bit-exact primitives, then A/B timings (FHEON_BCONV_TC=0/1)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_primitives.py -q -x 2>&1 | tail -3
for v in 1 0; do
  export FHEON_BCONV_TC=$v
  echo "== FHEON_BCONV_TC=$v"
  timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rot/s', d['value'], 'e2e', d['e2e']['value'])"
  timeout 300 python scripts/warm_probe.py 12 3 2>&1 | tail -1 | cut -c1-30
  timeout 400 python scripts/warm_probe.py 25 3 2>&1 | tail -1 | cut -c1-30
done
