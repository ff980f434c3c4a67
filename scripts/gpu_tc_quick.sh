#!/bin/bash
# bit-exact primitives + launch list of the timed bench steps
timeout 600 python -m pytest tests/test_gpu_primitives.py -q -x 2>&1 | tail -1
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline"
FHEON_PROFILE_RANGE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv $CMD > /dev/null 2>&1
python scripts/ncu_by_kernel.py gpurun_out/tc_launches.csv
