"""Where does ResNet-20's global_avg_pool time go? Per-layer timings over two
layer-timed inferences plus the isolated layer at its input level."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


depth = int(sys.argv[1]) if len(sys.argv) > 1 else 25
spec = M.resnet20(ring=65536, depth_budget=depth)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                      for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
em.infer(x)
for rep in range(2):
    r = em.infer(x, time_layers=True)
    top = sorted(r.layer_ms.items(), key=lambda kv: -kv[1])[:6]
    print("rep", rep, [(k, round(v, 1)) for k, v in top], flush=True)
for e in r.ledger[-8:]:
    print(e, flush=True)
ctx = em.ctx
for lv in (26, 14, 3):
    v = fh.SlotVector.encode(ctx, np.random.default_rng(1).uniform(-1, 1, 4096))
    v = fh.level_down(v, lv)
    fh.global_avg_pool(fh.PackedTensor(v, 64, 8))
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(3):
        fh.global_avg_pool(fh.PackedTensor(v, 64, 8))
    ctx.sync()
    print("global_avg_pool at limbs", lv, (time.perf_counter() - t0) / 3 * 1e3, "ms", flush=True)
