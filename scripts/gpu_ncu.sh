# Launch list of one timed headline step (encrypted ResNet-20, 128-bit chain) and a
# full capture of the top kernel families from the middle of it (one GPU, short run);
# the plain run of the same command line exits 0 first.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --quick --no-cpu-baseline --in-flight 1"
# (one image in flight: ncu serialises every launch, and host threads feeding several
# streams under it stall)
$CMD > gpurun_out/plain.log 2>&1 && \
FHEON_PROFILE_RANGE=1 timeout ${NCU_TIMEOUT:-900} ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo list rc=$?
FHEON_PROFILE_RANGE=1 timeout ${NCU_TIMEOUT:-900} ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"ntt_phase_kernel|k_ks_inner_sum|k_bconv_tc|k_mac" --launch-skip ${SKIP:-6000} -c ${COUNT:-16} \
  -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
tail -3 gpurun_out/ncu_full.log
python scripts/ncu_by_kernel.py gpurun_out/launches.csv | head -30
python scripts/ncu_table.py gpurun_out/prof_full.ncu-rep > gpurun_out/ncu_full.csv
