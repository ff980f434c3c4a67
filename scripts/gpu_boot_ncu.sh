#!/bin/bash
# ncu --set full of the bootstrap's non-NTT top kernels (ResNet-20 N=2^16 depth 25):
# the plain run of the same command exits 0 first
mkdir -p gpurun_out
CMD="python scripts/layer_profile.py bootstrap 25 25"
timeout 300 $CMD > gpurun_out/bn_plain.log 2>&1 || { echo "plain failed"; cat gpurun_out/bn_plain.log; exit 1; }
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_ks_inner_sum|k_mac|k_bconv_tc|k_tensor" -c 12 -o gpurun_out/boot_full $CMD > gpurun_out/bn_ncu.log 2>&1
echo ncu rc=$?
python scripts/ncu_table.py gpurun_out/boot_full.ncu-rep > gpurun_out/boot_full.csv 2>&1
cat gpurun_out/boot_full.csv
