# launch list + full capture of the top kernels (one GPU, short run); the plain
# run of the same command line exits 0 first
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo list rc=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ntt_phase_kernel|k_ks_inner|k_modup_bconv|k_moddown_conv|k_mac" -s 40 -c 10 -o gpurun_out/prof_r1b $CMD > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
tail -3 gpurun_out/ncu_full.log
