"""s/image of one model configuration (quick A/B on the GPU box):
  python scripts/model_time.py resnet20 12 128   (model, depth budget, security bits; 0 = insecure chain)"""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M

which = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 12
security = int(sys.argv[3]) if len(sys.argv) > 3 else 128
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3


def norm(x):
    return (x - 0.5) / 0.2887


if which == "resnet20":
    spec = M.resnet20(ring=65536, depth_budget=depth)
    spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                          for i in range(6)])
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
elif which == "vgg16":
    spec = M.calibrate_relu_scales(M.vgg16_paper(ring=65536, depth_budget=depth),
                                   [norm(np.random.default_rng(5002 + i).uniform(0, 1, (3, 32, 32))) for i in range(4)])
    x = norm(np.random.default_rng(5001).uniform(0, 1, (3, 32, 32)))
else:
    ring = int(sys.argv[5]) if len(sys.argv) > 5 else 32768
    spec = M.lenet5(ring=ring, depth_budget=depth)
    x = np.random.default_rng(3001).uniform(0, 1, (1, 28, 28))
t0 = time.perf_counter()
em = M.EncryptedModel(spec, security=security)
print("context", round(time.perf_counter() - t0, 2), "s", em.security, "L", em.ctx.L, "K", em.ctx.K, "dnum",
      em.ctx.dnum, "boots", em.n_boot, flush=True)
for _ in range(2):
    em.infer(x)
ts = []
for _ in range(reps):
    r = em.infer(x)
    ts.append(r.wall_ms / 1e3)
print(which, depth, security, "s/image", [round(t, 4) for t in ts], "median", round(float(np.median(ts)), 4),
      "key bytes", em.ctx.key_bytes(), r.stats, flush=True)
