set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.is_available())"
timeout 900 python -m pytest tests/test_gpu_primitives.py -x -q -m gpu 2>&1 | tail -30
