# ncu --set full of NTT phase launches from the middle of one headline step (one image, one
# stream: ncu serialises launches), after the same command exits 0 without ncu.  The report
# itself is too large for gpurun_out (64 MiB): the per-launch table and the source page are kept.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 2 --quick --no-cpu-baseline --no-rotations --in-flight 1 --image-batch 1"
$CMD > gpurun_out/plain.log 2>&1 && \
FHEON_PROFILE_RANGE=1 timeout ${NCU_TIMEOUT:-900} ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"ntt_phase_kernel" --launch-skip ${SKIP:-3000} -c ${COUNT:-32} \
  -o /tmp/prof_ntt $CMD > gpurun_out/ncu_ntt.log 2>&1
echo full rc=$?
tail -3 gpurun_out/ncu_ntt.log
python scripts/ncu_ntt_traffic.py /tmp/prof_ntt.ncu-rep > gpurun_out/ncu_resnet_ntt.csv
tail -1 gpurun_out/ncu_resnet_ntt.csv
