"""Host cost per engine call / per kernel launch at a tiny ring (GPU time negligible):
separates the C++ host path from device work (diagnostic)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh

cfg = fh.ContextConfig(1024, 512, 5, fh.CryptoMetadata(50, 40, 3), limbs=6, special_limbs=2, allow_insecure=True)
ctx = fh.SlotContext(cfg)
x = fh.SlotVector.encode(ctx, np.ones(512))
y = fh.SlotVector.encode(ctx, np.ones(512) * 2)
fh.rotate(x, 1)
for name, fn in (("add", lambda: fh.add(x, y)), ("rotate", lambda: fh.rotate(x, 1)),
                 ("mult_cipher", lambda: fh.mult_cipher(x, y)), ("rescale", lambda: fh.rescale(x))):
    fn()
    ctx.sync()
    s0 = ctx.stats()["launches"]
    t0 = time.perf_counter()
    n = 2000
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    ctx.sync()
    t2 = time.perf_counter()
    launches = (ctx.stats()["launches"] - s0) / n
    print(f"{name:12s} host {1e6 * (t1 - t0) / n:7.1f} us/call, {launches:.1f} launches/call -> "
          f"{1e6 * (t1 - t0) / n / max(launches, 1):6.1f} us/launch; drain {1e3 * (t2 - t1):.1f} ms", flush=True)
