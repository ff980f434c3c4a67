"""Stage-wise bootstrapping noise at N = 2^16, dense (sparse-secret encapsulation)
vs sparse main secret on the same chain and inputs (diagnostic)."""
import dataclasses
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import api, model as M

spec = M.resnet20(ring=65536, depth_budget=12)
base = M.ckks_config(spec, True, security=0)
cfgs = {"sparse": base, "dense": dataclasses.replace(base, hamming_weight=0)}
rng = np.random.default_rng(5)
S = 32768
z = rng.uniform(-1, 1, S)
u = rng.uniform(-0.95, 0.95, S)
w = rng.uniform(-1, 1, S) * 1e-3
out = {}
for name, cfg in cfgs.items():
    ctx = fh.SlotContext(cfg)
    L = ctx.L
    q0 = float(ctx.primes[0])
    r = {}
    x0 = fh.level_down(fh.SlotVector.encode(ctx, z), 1)
    r["level0_err"] = float(np.abs(x0.slots() - z).max())
    xt = fh.SlotVector.encode_top(ctx, z * q0 / ctx.scales[-1])
    r["cts"] = api.bootstrap_stage(xt, 1).slots_complex()
    xe = fh.level_down(fh.SlotVector.encode_top(ctx, u), L - 3)
    e = api.bootstrap_stage(xe, 2).slots()
    r["evalmod_err"] = float(np.abs(e - np.sin(2 * np.pi * 17.0 * u)).max())
    r["stc"] = api.bootstrap_stage(fh.SlotVector.encode_top(ctx, w), 3).slots_complex()
    y = fh.bootstrap(x0)
    r["boot_err"] = float(np.abs(y.slots() - z).max())
    # re-encrypt-free refresh twice
    y2 = fh.bootstrap(fh.level_down(y, 1))
    r["boot2_err"] = float(np.abs(y2.slots() - z).max())
    out[name] = r
    print(name, {k: v for k, v in r.items() if not isinstance(v, np.ndarray)}, flush=True)
    del ctx
print("cts dense-sparse max", np.abs(out["dense"]["cts"] - out["sparse"]["cts"]).max(),
      "cts magnitude", np.abs(out["sparse"]["cts"]).max())
print("stc dense-sparse max", np.abs(out["dense"]["stc"] - out["sparse"]["stc"]).max(),
      "stc magnitude", np.abs(out["sparse"]["stc"]).max())
