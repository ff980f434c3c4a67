set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layers.py tests/test_gpu_keys_client_server.py -x -q -m gpu 2>&1 | tail -3
for rep in 1 2; do
  timeout 900 python bench.py --quick --no-cpu-baseline --no-rotations > gpurun_out/bq_$rep.log 2> gpurun_out/bq_$rep.err; echo rc=$?
  tail -2 gpurun_out/bq_$rep.err
  python - <<P
import json
d=json.loads(open("gpurun_out/bq_$rep.log").read().strip().splitlines()[-1])
print("$rep", {k:d[k] for k in ("value","latency_s_per_image","ms_per_step")}, "e2e", d["e2e"]["value"])
P
done
timeout 900 python bench.py --quick --no-cpu-baseline --no-rotations --in-flight 3 > gpurun_out/bq_3.log 2> gpurun_out/bq_3.err; echo rc=$?
python - <<P
import json
d=json.loads(open("gpurun_out/bq_3.log").read().strip().splitlines()[-1])
print("F3", {k:d[k] for k in ("value","latency_s_per_image","ms_per_step")}, "e2e", d["e2e"]["value"])
P
nvidia-smi --query-gpu=memory.used --format=csv
