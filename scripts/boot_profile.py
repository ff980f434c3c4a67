"""One sparse-slot bootstrap (n = argv[1], default 4096) on the 128-bit ResNet-20
chain, for an ncu launch list of one stage: run with FHEON_BOOT_PROFILE=cos under
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ..."""
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
spec = M.resnet20(ring=65536, depth_budget=11)
ctx = fh.SlotContext(M.ckks_config(spec, True))
v = np.random.default_rng(3).uniform(-1, 1, 32768)
x = fh.level_down(fh.SlotVector.encode(ctx, v), 2)
y = fh.bootstrap(x, n)
ctx.sync()
print("err", float(np.abs(y.slots()[:n] - v[:n]).max()))
