"""Bootstrapping precision at N = 2^16 under chain / secret variants (diagnostic):
max |bootstrap(x) - x| over all slots, x uniform in [-1, 1]."""
import dataclasses
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

spec = M.resnet20(ring=65536, depth_budget=int(sys.argv[1]) if len(sys.argv) > 1 else 12)
sec = M.ckks_config(spec, True)
ins = M.ckks_config(spec, True, security=0)
variants = {
    "secure (dense+SSE, K=%d dnum=%d)" % (sec.special_limbs, sec.crypto.key_switch_digits): sec,
    "secure chain, sparse main h=64": dataclasses.replace(sec, hamming_weight=64, allow_insecure=True),
    "insecure (sparse h=64, K=%d dnum=3)" % ins.special_limbs: ins,
    "insecure chain, dense+SSE": dataclasses.replace(ins, hamming_weight=0),
    "secure chain, dense+SSE h_b=32": dataclasses.replace(sec, boot_hamming_weight=32),
}
for name, cfg in variants.items():
    ctx = fh.SlotContext(cfg)
    errs = []
    for s in range(3):
        v = np.random.default_rng(31 + s).uniform(-1, 1, ctx.slots())
        y = fh.bootstrap(fh.level_down(fh.SlotVector.encode(ctx, v), 1))
        errs.append(float(np.abs(y.slots() - v).max()))
    print(f"{name:45s} max err {max(errs):.3e}  {errs}", flush=True)
    del ctx
