set -x
mkdir -p gpurun_out
export FHEON_LIB_OVERRIDE=paper_2510_03996_b200/_lib/checked/libfheon_b200.so
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -6 > gpurun_out/checked_tests.log
cat gpurun_out/checked_tests.log
