set -x
mkdir -p gpurun_out
for B in 1 4; do
FHEON_BOOT_PROFILE=all ACTIVES=4096 REPS=1 timeout 1200 ncu --profile-from-start off --set full --clock-control none \
  -k regex:"k_ks_inner_sum|k_mac_bsgs" --launch-skip 3 -c 5 -o /tmp/prof_b$B python scripts/boot_batch_time.py $B > gpurun_out/ncu_b$B.log 2>&1
echo rc=$?
python scripts/ncu_kernel_traffic.py /tmp/prof_b$B.ncu-rep > gpurun_out/ncu_boot_batch_b$B.csv
cat gpurun_out/ncu_boot_batch_b$B.csv
done
