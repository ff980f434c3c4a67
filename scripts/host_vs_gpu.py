"""Is the single-image forward host- or GPU-bound?  Time until forward() returns
(host enqueue) vs until the stream drains; a GPU-bound run leaves tens of ms of
queued work at return (the launch queue holds ~1k launches), a host-bound one < 1 ms."""
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
for _ in range(4):
    em.forward(xin)
em.ctx.sync()
for _ in range(5):
    t0 = time.perf_counter()
    c0 = time.process_time()
    em.forward(xin)
    t1 = time.perf_counter()
    c1 = time.process_time()
    em.ctx.sync()
    t2 = time.perf_counter()
    print(f"enqueue {1e3 * (t1 - t0):.1f} ms (cpu {1e3 * (c1 - c0):.1f}), drain after return {1e3 * (t2 - t1):.1f} ms, "
          f"total {1e3 * (t2 - t0):.1f} ms", flush=True)
