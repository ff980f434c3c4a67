import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import api
logN = int(sys.argv[1]) if len(sys.argv) > 1 else 12
L = int(sys.argv[2]) if len(sys.argv) > 2 else 24
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
N = 1 << logN; S = N // 2
cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=L, special_limbs=K, special_bits=60, seed=5,
                       hamming_weight=64, bootstrap=True, boot_scale_bits=55)
t0 = time.time()
ctx = fh.SlotContext(cfg)
info = api.bootstrap_info(ctx)
print(f"N=2^{logN} L={L}: setup {time.time()-t0:.2f}s keys {ctx.key_count()} depth {info['depth']} budget {ctx.depth_budget()} cos deg {len(info['cos_coeffs'])-1}")
print("primes bits", [int(q).bit_length() for q in ctx.primes], "T bits", [round(float(np.log2(t)), 2) for t in ctx.scales], flush=True)
rng = np.random.default_rng(1)
for mag in (1.0, 4.0, 8.0):
    v = rng.uniform(-mag, mag, S)
    x = fh.SlotVector.encode(ctx, v)
    x0 = fh.level_down(x, 1)
    ctx.sync(); t1 = time.time()
    y = fh.bootstrap(x0)
    ctx.sync(); dt = time.time() - t1
    d = y.slots()
    print(f"mag {mag}: level {x.level()} -> 0 -> boot {y.level()}: max err {np.abs(d - v).max():.3e} mean {np.abs(d-v).mean():.3e} time {dt*1e3:.1f} ms", flush=True)
