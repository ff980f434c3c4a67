mkdir -p gpurun_out
timeout 300 python scripts/host_vs_gpu.py > gpurun_out/hvg.log 2>&1; cat gpurun_out/hvg.log | tail -6
FHEON_SECURITY=128 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/mp_r20_128.csv python scripts/model_profile.py resnet20 11 > gpurun_out/mp_ncu.log 2>&1 || echo "ncu failed"
tail -2 gpurun_out/mp_ncu.log
python scripts/ncu_by_kernel.py gpurun_out/mp_r20_128.csv
python scripts/ntt_buckets.py gpurun_out/mp_r20_128.csv
