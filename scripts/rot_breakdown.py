import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_03996_b200 as fh
ctx = fh.SlotContext(fh.ContextConfig.preset("config2"))
steps = [1 << i for i in range(15)] + [-1]
ctx.keygen_rotations(steps)
rng = np.random.default_rng(0)
cts = [fh.SlotVector.encode_top(ctx, rng.uniform(-1, 1, 32768)) for _ in range(8)]
stream = torch.cuda.ExternalStream(ctx.stream())
def run(n):
    c = 0
    for s in range(n):
        fh.rotate_many(cts, [steps[(c + b) % 16] for b in range(8)]); c += 8
run(3); ctx.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream); run(20); e1.record(stream); e1.synchronize()
tot = e0.elapsed_time(e1) / 20
print(f"step {tot:.3f} ms (8 rotations) = {tot/8*1e3:.1f} us/rotation")
for cls, name in ((2, "ntt"), (1, "ks_inner"), (3, "modup_bconv"), (4, "moddown_conv")):
    ctx.timer_arm(cls); run(20); ms, n = ctx.timer_read(); ctx.timer_arm(0)
    print(f"  {name:14s} {ms/20:.3f} ms/step ({100*ms/20/tot:.0f}%)  scopes/step {n/20:.0f}")
st0 = ctx.stats(); run(1); st1 = ctx.stats()
print("launches per step", st1["launches"] - st0["launches"], "ntt limbs per step", st1["ntt_limbs"] - st0["ntt_limbs"])
