"""Bootstrapping transform-level split (CoeffsToSlots, SlotsToCoeffs) on the 128-bit
ResNet-20 chain: chain shape, bootstrap time / error and s/image (diagnostic)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 11
cts, stc = int(sys.argv[2]), int(sys.argv[3])


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=depth),
                               [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
cfg = M.ckks_config(spec, True, boot_levels=(cts, stc))
ctx = fh.SlotContext(cfg)
S = ctx.slots()
v = np.random.default_rng(1).uniform(-1, 1, S)
x0 = fh.level_down(fh.SlotVector.encode(ctx, v), 1)
fh.bootstrap(x0)
ctx.sync()
t0 = time.perf_counter()
for _ in range(5):
    y = fh.bootstrap(x0)
ctx.sync()
bt = (time.perf_counter() - t0) / 5 * 1e3
err = float(np.abs(y.slots() - v).max())
print(f"cts {cts} stc {stc}: L {cfg.limbs} K {cfg.special_limbs} dnum {cfg.crypto.key_switch_digits} "
      f"logQP {fh.host_security(cfg)['log2_qp']} boot {bt:.2f} ms err {err:.2e}", flush=True)
em = M.EncryptedModel(spec, boot_levels=(cts, stc))
xin = em.encrypt_input(x)
for _ in range(2):
    em.forward(xin)
em.ctx.sync()
t0 = time.perf_counter()
for _ in range(3):
    o = em.forward(xin)
em.ctx.sync()
st = (time.perf_counter() - t0) / 3
from oracle import ref as sref
import tempfile
rl, _, _, _ = sref.infer(spec.write(tempfile.mkdtemp()), x)
print(f"   resnet20 d{depth} {st:.4f} s/image, logit err vs reference {np.abs(o.slots()[:10] - rl).max():.2e}",
      flush=True)
