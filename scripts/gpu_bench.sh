set -x
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$?
tail -3 gpurun_out/bench.err
cut -c1-400 gpurun_out/bench.log
