"""Per-inference op counts during warm-up (ResNet-20, N=2^16): what is still
being built on the second inference?"""
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
em = M.EncryptedModel(M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=depth), cal))
import subprocess
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    em.ctx.timer_arm(2)
    t0 = time.perf_counter()
    r = em.infer(x, time_layers=(i == 1))
    wall = time.perf_counter() - t0
    ntt_ms, _ = em.ctx.timer_read()
    em.ctx.timer_arm(0)
    smi = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,memory.used,clocks_throttle_reasons.active",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(i, round(wall, 3), "ntt_ms", round(ntt_ms), {k: r.stats[k] for k in ("encodes", "launches")},
          "keys", em.ctx.key_count(), smi, flush=True)
    if i == 1:
        top = sorted(r.layer_ms.items(), key=lambda kv: -kv[1])[:8]
        print("   slowest layers", [(k, round(v)) for k, v in top])
