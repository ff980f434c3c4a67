set -x
mkdir -p gpurun_out
for mode in noclk 2000 500; do
  if [ $mode = noclk ]; then export FHEON_NO_CLOCKS=1; else unset FHEON_NO_CLOCKS; export FHEON_CLOCKS_MS=$mode; fi
  timeout 900 python bench.py --quick --no-cpu-baseline --no-rotations > gpurun_out/bq_$mode.log 2> gpurun_out/bq_$mode.err; echo rc=$?
  python - <<P
import json
d=json.loads(open("gpurun_out/bq_$mode.log").read().strip().splitlines()[-1])
print("$mode", {k:d[k] for k in ("value","latency_s_per_image","ms_per_step")}, "e2e", d["e2e"]["value"], d["clocks"])
P
done
