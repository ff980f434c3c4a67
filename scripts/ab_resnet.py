"""ResNet-20 128-bit forward s/image (median of 6 after 3 warm-ups) for A/B of engine builds."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.resnet20(ring=65536, depth_budget=11)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                      for i in range(3)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
xin = em.encrypt_input(x)
for _ in range(3):
    em.forward(xin)
em.ctx.sync()
ts = []
for _ in range(6):
    t = time.perf_counter()
    em.forward(xin)
    em.ctx.sync()
    ts.append(time.perf_counter() - t)
print(sys.argv[1] if len(sys.argv) > 1 else "", "resnet20 s/image", round(float(np.median(ts)), 4), [round(v, 4) for v in ts])
