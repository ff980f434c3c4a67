# launch list of the timed bench steps + a full capture of the top kernels
# (one GPU, short run); the plain run of the same command line exits 0 first
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
FHEON_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo list rc=$?
FHEON_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"ntt_phase_kernel|k_ks_inner|k_bconv_tc" -c 10 -o gpurun_out/prof_r1f $CMD \
  > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
tail -3 gpurun_out/ncu_full.log
python scripts/ncu_by_kernel.py gpurun_out/launches.csv
