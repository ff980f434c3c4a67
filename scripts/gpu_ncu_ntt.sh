set -x
mkdir -p gpurun_out
python scripts/prof_prims.py 0 > gpurun_out/plain_ntt.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ntt_phase_kernel -s 4 -c 2 -o gpurun_out/prof_ntt python scripts/prof_prims.py 0 > gpurun_out/ncu_ntt.log 2>&1
echo rc=$?
