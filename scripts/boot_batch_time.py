"""bootstrap_many on the 128-bit ResNet-20 chain: ms per ciphertext for batches of B
(active = S/2, S/4, S/8; clean inputs at level 0 like the network's).  FHEON_BOOT_TIMING=1
adds the per-stage laps (synchronising)."""
import os
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

spec = M.resnet20(ring=65536, depth_budget=11)
ctx = fh.SlotContext(M.ckks_config(spec, True))
S = 32768
rng = np.random.default_rng(3)
Bs = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
REPS = int(os.environ.get("REPS", "4"))
for active in [int(a) for a in os.environ.get("ACTIVES", f"{S // 2},{S // 8}").split(",")]:
    vs = []
    for _ in range(max(Bs)):
        v = rng.uniform(-1, 1, S)
        v[active:] = 0.0
        vs.append(v)
    xs = [fh.level_down(fh.SlotVector.encode(ctx, v), 1) for v in vs]
    for B in Bs:
        fh.bootstrap_many(xs[:B], active, clean=True)
        ctx.sync()
        ts = []
        for _ in range(REPS):
            t = time.perf_counter()
            ys = fh.bootstrap_many(xs[:B], active, clean=True)
            ctx.sync()
            ts.append(time.perf_counter() - t)
        err = max(float(np.abs(y.slots()[:active] - v[:active]).max()) for y, v in zip(ys, vs))
        print(f"active {active} B={B}: {1e3 * float(np.median(ts)) / B:.3f} ms per ciphertext "
              f"({1e3 * float(np.median(ts)):.2f} ms per batch), err {err:.2e}", flush=True)
        del ys
