#!/bin/bash
# kernel-level breakdown of ResNet-20 blocks (see scripts/layer_profile.py)
mkdir -p gpurun_out
for b in ${BLOCKS:-conv2 conv3 relu bootstrap}; do
  timeout 300 python scripts/layer_profile.py $b ${DEPTH:-12} > gpurun_out/lp_$b.plain 2>&1 || echo "plain $b failed"
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/lp_$b.csv python scripts/layer_profile.py $b ${DEPTH:-12} ${DEPTH:-12} > gpurun_out/lp_$b.log 2>&1 || echo "ncu $b failed"
  echo "== $b"; tail -1 gpurun_out/lp_$b.plain; python scripts/ncu_by_kernel.py gpurun_out/lp_$b.csv
done
