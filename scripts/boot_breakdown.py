"""Device time and op counts of each bootstrapping stage at the ResNet-20
parameters (N=2^16, depth budget 12, 29 limbs): ModRaise, CoeffsToSlots
(incl. conjugation split), EvalMod (two real halves), SlotsToCoeffs."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import api
from paper_2510_03996_b200 import model as M

ring = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 12
spec = M.resnet20(ring=ring, depth_budget=depth)
ctx = fh.SlotContext(M.ckks_config(spec, True))
info = api.bootstrap_info(ctx)
S = ring // 2
v = np.random.default_rng(1).uniform(-1, 1, S)
x = fh.level_down(fh.SlotVector.encode(ctx, v), 1)
fh.bootstrap(x)  # warm (plaintext caches, allocator)
ctx.sync()


def timed(fn, reps=3):
    ctx.reset_stats()
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    ctx.sync()
    dt = (time.perf_counter() - t0) / reps * 1e3
    st = {k: v // reps for k, v in ctx.stats().items()}
    return out, dt, st


raised, t_mr, s_mr = timed(lambda: api.bootstrap_stage(x, 4))
cts, t_cts, s_cts = timed(lambda: api.bootstrap_stage(raised, 1))
em_in = fh.level_down(cts, cts.level() + 1)
em, t_em, s_em = timed(lambda: api.bootstrap_stage(em_in, 2))
stc, t_stc, s_stc = timed(lambda: api.bootstrap_stage(em, 3))
full, t_full, s_full = timed(lambda: fh.bootstrap(x))
print(f"ring {ring} limbs {ctx.L} K {ctx.K} depth {info['depth']} cos degree {len(info['cos_coeffs']) - 1}")
for name, t, s in (("modraise", t_mr, s_mr), ("coeffs_to_slots", t_cts, s_cts), ("evalmod(1 half)", t_em, s_em),
                   ("slots_to_coeffs", t_stc, s_stc), ("full bootstrap", t_full, s_full)):
    print(f"  {name:18s} {t:8.2f} ms  ks {s['keyswitches']:4d} rot {s['rotations']:4d} mc {s['mult_cipher']:3d} "
          f"mp {s['mult_plain']:4d} resc {s['rescales']:4d} ntt_limbs {s['ntt_limbs']:6d} launches {s['launches']}")
print(f"  levels: raised {raised.level()} cts {cts.level()} evalmod {em.level()} stc {stc.level()} full {full.level()}")
err = np.abs(full.slots() - v).max()
print(f"  bootstrap max err {err:.2e}")
