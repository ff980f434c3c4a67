import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M
spec = M.resnet20(ring=65536, depth_budget=25)
ctx = fh.SlotContext(M.ckks_config(spec, True))
v = np.random.default_rng(1).uniform(-1, 1, 32768)
x = fh.level_down(fh.SlotVector.encode(ctx, v), 1)
for i in range(6):
    ctx.sync(); t0 = time.perf_counter(); y = fh.bootstrap(x); ctx.sync()
    print(i, (time.perf_counter() - t0) * 1e3, "ms", flush=True)
