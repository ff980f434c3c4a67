"""Bootstrap time per variant on the 128-bit ResNet-20 chain (N=2^16, depth 11):
full vs sparse-slot (active = S/2, S/4, S/8), max error over the kept slots,
then one ResNet-20 inference (s/image).  Device-synchronised wall clock after warm-up."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

spec = M.resnet20(ring=65536, depth_budget=11)
t0 = time.perf_counter()
ctx = fh.SlotContext(M.ckks_config(spec, True))
print("context_s", round(time.perf_counter() - t0, 2), "keys", ctx.key_count(), flush=True)
S = 32768
rng = np.random.default_rng(3)
v = rng.uniform(-1, 1, S)
x = fh.level_down(fh.SlotVector.encode(ctx, v), 2)
for active in (None, S // 2, S // 4, S // 8):
    fh.bootstrap(x, active)
    ctx.sync()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        y = fh.bootstrap(x, active)
        ctx.sync()
        ts.append(time.perf_counter() - t)
    a = active or S
    err = float(np.abs(y.slots()[:a] - v[:a]).max())
    print("bootstrap active", a, "ms", round(1e3 * float(np.median(ts)), 3), "err", f"{err:.2e}", flush=True)
del ctx
if len(sys.argv) > 1:
    def norm(x):
        return (x - 0.5) / 0.2887
    spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                          for i in range(6)])
    xi = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
    for sp in (0, 3):
        em = M.EncryptedModel(spec, boot_sparse=sp)
        xin = em.encrypt_input(xi)
        for _ in range(2):
            o = em.forward(xin)
        em.ctx.sync()
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            o = em.forward(xin)
            em.ctx.sync()
            ts.append(time.perf_counter() - t)
        print("resnet20 boot_sparse", sp, "s/image", round(float(np.median(ts)), 4), "logits", np.round(o.slots()[:10], 5),
              flush=True)
        del em
