"""NTT time per limb-poly vs batch size (N=2^16), device time via the microbench."""
import sys
sys.path.insert(0, '.')
import paper_2510_03996_b200 as fh
ctx = fh.SlotContext(fh.ContextConfig.preset('config2'))
for batch, limbs in ((1, 2), (1, 4), (1, 8), (1, 12), (1, 24), (2, 24), (4, 24), (8, 24), (16, 24)):
    for k, name in ((0, "ntt"), (1, "intt")):
        ms = min(ctx.microbench(k, batch, limbs, 8, 50) for _ in range(3))
        polys = batch * limbs * 2
        print(f"{name} {polys:4d} limb-polys: {ms * 1e3:8.1f} us per call, {ms * 1e3 / polys:6.3f} us per limb-poly")
