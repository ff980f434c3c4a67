"""Per-layer-type wall time (device-synchronised after every layer) of one
128-bit ResNet-20 inference (N=2^16, depth 11), summed by type; residual units
are split into their children (the unit row itself is the skip add)."""
import collections
import sys

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.resnet20(ring=65536, depth_budget=int(sys.argv[1]) if len(sys.argv) > 1 else 11)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                      for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
for _ in range(2):
    em.infer(x)
r = em.infer(x, time_layers=True)
names = {}


def walk(layers):
    for b in layers:
        names[b.name] = b.type
        if b.type == "residual":
            walk(b.body)
            walk(b.downsample)


walk(em.layers)
agg = collections.defaultdict(float)
cnt = collections.Counter()
for n, t in r.layer_ms.items():
    agg[names.get(n, n)] += t
    cnt[names.get(n, n)] += 1
# residual rows include their children: subtract
res = sum(t for n, t in r.layer_ms.items() if names.get(n) == "residual")
child = 0.0
for b in em.layers:
    if b.type == "residual":
        for c in list(b.body) + list(b.downsample):
            child += r.layer_ms.get(c.name, 0.0)
agg["residual"] = res - child
tot = sum(v for k, v in agg.items())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{k:20s} {v:9.2f} ms  n={cnt[k]:3d}  {100 * v / tot:5.1f}%")
print("total", round(tot, 1), "ms")
