import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M
import paper_2510_03996_b200 as fh
def norm(x): return (x - 0.5) / 0.2887
spec = M.resnet20(ring=65536, depth_budget=12)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
em.infer(x)
# host enqueue time vs device time: run the layer loop without the final decrypt
for rep in range(2):
    em.ctx.sync()
    t0 = time.perf_counter()
    v = fh.SlotVector.encode(em.ctx, x.reshape(-1))
    for b in em.layers:
        v = em._run(b, v, None)
    th = time.perf_counter() - t0
    em.ctx.sync()
    tw = time.perf_counter() - t0
    print(f"host enqueue {th:.2f}s, wall incl. device drain {tw:.2f}s", flush=True)
# per kernel class device time (live CUDA events)
for cls, name in ((2, "ntt"), (1, "ks_inner"), (3, "modup_bconv"), (4, "moddown_conv")):
    em.ctx.timer_arm(cls)
    em.infer(x)
    ms, n = em.ctx.timer_read()
    em.ctx.timer_arm(0)
    print(f"{name}: {ms:.0f} ms over {n} scopes", flush=True)
