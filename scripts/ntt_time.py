"""NTT / iNTT device time per limb at config2 (N=2^16), batch of 8 ciphertexts x 24 limbs x 2 polys."""
import sys
sys.path.insert(0, '.')
import paper_2510_03996_b200 as fh
ctx = fh.SlotContext(fh.ContextConfig.preset('config2'))
for k, name in ((0, "ntt"), (1, "intt")):
    ms = min(ctx.microbench(k, 8, 24, 8, 20) for _ in range(3))
    print(f"{name}: {ms / 8:.4f} ms per ciphertext (48 limb-polys), {ms / 8 / 48 * 1e3:.3f} us per limb")
