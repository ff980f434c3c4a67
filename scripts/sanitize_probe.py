"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
the smoke path (rotation, encrypted conv), a relinearised product, rotate-and-sum,
packed async transfers on the copy streams, and one full bootstrap -- at N = 2^12
so every kernel family runs (NTT phases, k_ks_inner*, k_bconv_tc warp-specialised
tcgen05 basis conversion, k_mac, pack/unpack) in a few seconds under the tools."""
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh

N, S = 1 << 12, 1 << 11
cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=24, special_limbs=8, special_bits=60, seed=5,
                       bootstrap=True, boot_scale_bits=55, allow_insecure=True)
ctx = fh.SlotContext(cfg)
rng = np.random.default_rng(1)
v = rng.uniform(-1, 1, S)
x = fh.SlotVector.encode(ctx, v)
y = fh.rotate(x, 3)
z = fh.mult_cipher(x, y)
s = fh.rotate_sum([x, y], [1, -5])
h = fh.rotate_hoisted(x, [1, 2, 4, 8])
pk = x.packed()
xp = fh.SlotVector.from_packed(ctx, pk, x.limbs(), x.scale(), async_copy=True)
out = np.zeros_like(pk)
xp.packed(out=out, async_copy=True)
ctx.wait_transfers()
assert np.array_equal(out, pk)
w = rng.uniform(-1, 1, (3, 2, 3, 3))
c = fh.convolution(fh.PackedTensor(fh.SlotVector.encode(ctx, rng.uniform(-1, 1, 2 * 64)), 2, 8),
                   fh.ConvConfig(2, 3, 3, 1, 1, fh.ConvMode.special3x3), fh.KernelTensor(w))
b = fh.bootstrap(fh.level_down(x, 1))
err = float(np.abs(b.slots() - v).max())
assert err < 1e-4, err
print("sanitize probe ok", err, z.level(), s.level(), len(h), c.data.level())
