"""Host-side cost of one 128-bit ResNet-20 forward pass by layer type (cProfile over
the ctypes calls: their time is C++ host work, the forward pass never synchronises)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=11),
                               [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
xin = em.encrypt_input(x)
for _ in range(2):
    em.forward(xin)
em.ctx.sync()
t0 = time.perf_counter()
em.forward(xin)
t1 = time.perf_counter()
em.ctx.sync()
t2 = time.perf_counter()
print(f"host enqueue {1e3 * (t1 - t0):.1f} ms, device drain after {1e3 * (t2 - t1):.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
em.forward(xin)
pr.disable()
em.ctx.sync()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(12)
