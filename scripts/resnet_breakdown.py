"""Per-layer-type device time of encrypted ResNet-20 (N=2^16, depth 12) plus
kernel-class totals; used to pick the next optimisation target."""
import collections
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M

which = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def norm(x):
    return (x - 0.5) / 0.2887


if which == "resnet20":
    spec = M.resnet20(ring=65536, depth_budget=depth)
    spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                          for i in range(6)])
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
elif which == "vgg16":
    spec = M.calibrate_relu_scales(M.vgg16_paper(ring=65536, depth_budget=depth),
                                   [norm(np.random.default_rng(5002 + i).uniform(0, 1, (3, 32, 32))) for i in range(4)])
    x = norm(np.random.default_rng(5001).uniform(0, 1, (3, 32, 32)))
else:
    spec = M.lenet5(ring=32768, depth_budget=depth)
    x = np.random.default_rng(3001).uniform(0, 1, (1, 28, 28))
em = M.EncryptedModel(spec, security=int(__import__('os').environ.get('FHEON_SECURITY', '0')))
em.infer(x)
em.infer(x)
t0 = time.perf_counter()
r = em.infer(x)
print(f"{which}: {time.perf_counter() - t0:.3f} s/image", flush=True)
r = em.infer(x, time_layers=True)
kinds = {}


def walk(layers):
    for b in layers:
        kinds[b.name] = b.type if b.type != "conv" else f"conv{b.src.params['kernel']}"
        walk(getattr(b, "body", []) or [])
        walk(getattr(b, "downsample", []) or [])


walk(em.layers)
agg = collections.defaultdict(float)
cnt = collections.Counter()
for name, ms in r.layer_ms.items():
    k = kinds.get(name, "?")
    if k == "residual":
        continue  # contains its body
    agg[k] += ms
    cnt[k] += 1
tot = sum(agg.values())
for k, ms in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"  {k:18s} {ms:9.1f} ms  ({cnt[k]} calls, {100 * ms / tot:.1f}%)")
print(f"  total(layer-timed) {tot:.1f} ms; stats {r.stats}", flush=True)
for cls, name in ((2, "ntt"), (1, "ks_inner"), (3, "modup_bconv"), (4, "moddown_conv")):
    em.ctx.timer_arm(cls)
    em.infer(x)
    ms, n = em.ctx.timer_read()
    em.ctx.timer_arm(0)
    print(f"  class {name}: {ms:.0f} ms over {n} scopes", flush=True)
