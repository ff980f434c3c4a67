#!/bin/bash
# whole-inference kernel breakdown (scripts/model_profile.py) + layer-type split
mkdir -p gpurun_out
M=${MODEL:-resnet20}; D=${DEPTH:-25}
timeout 600 python scripts/resnet_breakdown.py $M $D > gpurun_out/mp_breakdown.log 2>&1 || echo "breakdown failed"
cat gpurun_out/mp_breakdown.log
timeout 300 python scripts/model_profile.py $M $D > gpurun_out/mp_plain.log 2>&1 || echo "plain failed"
cat gpurun_out/mp_plain.log
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/mp_${M}_d${D}.csv python scripts/model_profile.py $M $D > gpurun_out/mp_ncu.log 2>&1 || echo "ncu failed"
tail -2 gpurun_out/mp_ncu.log
python scripts/ncu_by_kernel.py gpurun_out/mp_${M}_d${D}.csv
