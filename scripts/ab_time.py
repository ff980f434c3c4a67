"""A/B timing probe (run once per library variant via FHEON_LIB_OVERRIDE): the
128-bit ResNet-20 headline s/image, configs[1] rotation throughput and a
bootstrap, all device-synchronised wall clock after warm-up."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

tag = sys.argv[1] if len(sys.argv) > 1 else "?"
what = sys.argv[2] if len(sys.argv) > 2 else "all"
out = {}
if what in ("all", "rot"):
    ctx = fh.SlotContext(fh.ContextConfig.preset("config2"))
    out["rot_ms"] = round(ctx.microbench(3, 8, 24, 1, 20) / 8, 4)
    out["hoist32_ms"] = round(ctx.microbench(4, 1, 24, 32, 5) / 32, 4)
    out["mac25_ms"] = round(ctx.microbench(9, 1, 24, 25, 20), 4)
    out["ntt_ms"] = round(ctx.microbench(0, 8, 24, 1, 20) / 8, 4)
    del ctx
if what in ("all", "resnet"):
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
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        o = em.forward(xin)
        em.ctx.sync()
        ts.append(time.perf_counter() - t0)
    out["resnet_s"] = round(float(np.median(ts)), 4)
    out["logit0"] = float(o.slots()[0])
print(tag, out, flush=True)
