#!/bin/bash
# ncu --set full of one bootstrap's top kernels on the headline's 128-bit chain
# (ResNet-20 N=2^16, depth 11): NTT phases, k_ks_inner_sum, k_mac, k_bconv_tc.
# The plain run of the same command exits 0 first.
mkdir -p gpurun_out
export FHEON_SECURITY=${FHEON_SECURITY:-128}
CMD="python scripts/layer_profile.py bootstrap ${DEPTH:-11}"
timeout 300 $CMD > gpurun_out/bn_plain.log 2>&1 || { echo "plain failed"; cat gpurun_out/bn_plain.log; exit 1; }
timeout ${NCU_TIMEOUT:-900} ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-ntt_phase_kernel|k_ks_inner_sum|k_mac|k_bconv_tc}" --launch-skip ${SKIP:-40} -c ${COUNT:-12} \
  -o gpurun_out/boot_full $CMD > gpurun_out/bn_ncu.log 2>&1
echo ncu rc=$?
tail -2 gpurun_out/bn_ncu.log
python scripts/ncu_table.py gpurun_out/boot_full.ncu-rep > gpurun_out/boot_full.csv 2>&1
cat gpurun_out/boot_full.csv
