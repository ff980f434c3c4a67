"""bootstrap max error at N = 2^16 (depth 12 chain): the 128-bit chain (dense secret,
sparse-secret encapsulation, 60-bit bootstrapping levels) vs the insecure sparse one,
for a few input magnitudes (diagnostic; env FHEON_BOOT_DEBUG etc. pass through)."""
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

spec = M.resnet20(ring=65536, depth_budget=int(sys.argv[1]) if len(sys.argv) > 1 else 12)
for name, cfg in {"secure": M.ckks_config(spec, True), "sparse": M.ckks_config(spec, True, security=0)}.items():
    ctx = fh.SlotContext(cfg)
    for mag in (1.0, 8.0, 0.0):
        v = np.random.default_rng(1).uniform(-1, 1, ctx.slots()) * mag
        y = fh.bootstrap(fh.level_down(fh.SlotVector.encode(ctx, v), 1))
        print(name, "mag", mag, "err", float(np.abs(y.slots() - v).max()), flush=True)
    del ctx
