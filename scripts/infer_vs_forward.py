import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M
def norm(x): return (x - 0.5) / 0.2887
spec = M.resnet20(ring=65536, depth_budget=11)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(3)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
xin = em.encrypt_input(x)
for _ in range(2): em.forward(xin)
em.ctx.sync()
t = time.perf_counter(); em.forward(xin); em.ctx.sync(); print("forward", time.perf_counter() - t, flush=True)
for k in range(3):
    t = time.perf_counter(); r = em.infer(x); print("infer", time.perf_counter() - t, r.wall_ms, flush=True)
t = time.perf_counter(); r = em.infer(x, time_layers=True); print("infer timed", time.perf_counter() - t, flush=True)
print(sorted(r.layer_ms.items(), key=lambda kv: -kv[1])[:8])
t = time.perf_counter(); em.forward(xin); em.ctx.sync(); print("forward", time.perf_counter() - t, flush=True)
