"""bootstrap max error at N = 2^16 (depth 12 chain) for chain variants (diagnostic):
boot_scale_bits x first-modulus bits, dense secret (sparse-secret encapsulation)."""
import dataclasses
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

base = M.ckks_config(M.resnet20(ring=65536, depth_budget=12), True, security=0)
for bb, q0 in [(55, 55), (58, 55), (60, 55), (60, 58), (60, 60)]:
    cfg = dataclasses.replace(base, hamming_weight=0, boot_scale_bits=bb,
                              crypto=dataclasses.replace(base.crypto, first_modulus_bits=q0), special_limbs=12)
    try:
        ctx = fh.SlotContext(cfg)
    except Exception as e:
        print(bb, q0, "ERR", e, flush=True)
        continue
    pb = [int(q).bit_length() for q in ctx.primes[:ctx.L]]
    errs = []
    for mag in (1.0, 8.0):
        v = np.random.default_rng(1).uniform(-1, 1, ctx.slots()) * mag
        y = fh.bootstrap(fh.level_down(fh.SlotVector.encode(ctx, v), 1))
        errs.append(float(np.abs(y.slots() - v).max()))
    print("boot_bits", bb, "q0", q0, "maxbits", max(pb), "logQ", round(float(np.log2(ctx.primes[:ctx.L].astype(float)).sum()), 1),
          "err(mag1, mag8)", errs, flush=True)
    del ctx
