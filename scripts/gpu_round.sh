# One GPU call of a round: smoke, the whole -m gpu suite, the default bench and the reference arm.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$?
tail -3 gpurun_out/bench.err
cut -c1-400 gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo rc=$?
cut -c1-300 gpurun_out/bench_ref.log
