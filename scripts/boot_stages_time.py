"""Device time of each bootstrapping stage on the 128-bit headline chain (diagnostic):
ModRaise (+ encapsulation switches), CoeffsToSlots, EvalMod (one half), SlotsToCoeffs,
and the whole bootstrap."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import api, model as M

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 11
ctx = fh.SlotContext(M.ckks_config(M.resnet20(ring=65536, depth_budget=depth), True))
S = ctx.slots()
v = np.random.default_rng(1).uniform(-1, 1, S)
x0 = fh.level_down(fh.SlotVector.encode(ctx, v), 1)
top = fh.SlotVector.encode_top(ctx, v * 1e-3)
L = ctx.L
xe = fh.level_down(fh.SlotVector.encode_top(ctx, v * 0.5), L - 3)


def timeit(fn, reps=5):
    fn()
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    ctx.sync()
    return (time.perf_counter() - t0) / reps * 1e3


print("modraise  %.2f ms" % timeit(lambda: api.bootstrap_stage(x0, 4)))
print("cts       %.2f ms" % timeit(lambda: api.bootstrap_stage(top, 1)))
print("evalmod/2 %.2f ms" % timeit(lambda: api.bootstrap_stage(xe, 2)))
print("stc       %.2f ms" % timeit(lambda: api.bootstrap_stage(top, 3)))
print("bootstrap %.2f ms" % timeit(lambda: fh.bootstrap(x0)))
print(api.bootstrap_info(ctx))
