"""ResNet-20 (N=2^16, depth 25) inference times vs the weight-plaintext cache budget."""
import gc
import subprocess
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


depth = int(sys.argv[1]) if len(sys.argv) > 1 else 25
cal = [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)]
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=depth), cal)
for gb in [int(v) for v in sys.argv[2:]] or [0, 16, 32, 64]:
    em = M.EncryptedModel(spec)
    em.ctx.set_weight_cache(gb << 30)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        em.infer(x)
        ts.append(round(time.perf_counter() - t0, 3))
    mem = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader"], capture_output=True,
                         text=True).stdout.strip()
    print(f"depth {depth} weight cache {gb} GiB: {ts}  {mem}", flush=True)
    del em
    gc.collect()
