set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bootstrap.py tests/test_gpu_models.py -x -q -m gpu -k "many or batch" 2>&1 | tail -15
timeout 600 python scripts/ab_batch.py 0 1 2 4 8 2>&1 | tail -8
FLIGHT=2 timeout 600 python scripts/ab_batch.py 2 4 2>&1 | tail -4
