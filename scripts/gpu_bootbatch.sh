set -x
mkdir -p gpurun_out
for B in 1 4; do
FHEON_BOOT_PROFILE=all ACTIVES=4096 REPS=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/boot_b$B.csv python scripts/boot_batch_time.py $B > gpurun_out/boot_b$B.log 2>&1 || echo "ncu failed"
tail -2 gpurun_out/boot_b$B.log
python scripts/ncu_by_kernel.py gpurun_out/boot_b$B.csv | head -24
python scripts/ntt_buckets.py gpurun_out/boot_b$B.csv
done
timeout 600 python scripts/ab_batch.py 4 8 2>&1 | tail -3
FLIGHT=2 timeout 600 python scripts/ab_batch.py 4 8 2>&1 | tail -3
FLIGHT=3 timeout 600 python scripts/ab_batch.py 2 4 2>&1 | tail -3
FLIGHT=4 timeout 600 python scripts/ab_batch.py 0 2 2>&1 | tail -3
