"""ResNet-20 128-bit forward s/image (median of 6 after 3 warm-ups) for A/B of engine builds."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.resnet20(ring=65536, depth_budget=11)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                      for i in range(3)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
xin = em.encrypt_input(x)
for _ in range(int(__import__("os").environ.get("WARM", "3"))):
    em.forward(xin)
em.ctx.sync()
ts = []


def pool_gb():
    try:
        from cuda import cudart
        _, pool = cudart.cudaDeviceGetDefaultMemPool(0)
        _, r = cudart.cudaMemPoolGetAttribute(pool, cudart.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
        _, u = cudart.cudaMemPoolGetAttribute(pool, cudart.cudaMemPoolAttr.cudaMemPoolAttrUsedMemHigh)
        return round(int(r) / 1e9, 2), round(int(u) / 1e9, 2)
    except Exception as e:  # noqa: BLE001
        return str(e)[:40]


for _ in range(int(__import__("os").environ.get("REPS", "6"))):
    t = time.perf_counter()
    em.forward(xin)
    em.ctx.sync()
    ts.append(time.perf_counter() - t)
    if __import__("os").environ.get("POOL"):
        print(round(ts[-1], 4), "pool reserved / used-high GB", pool_gb(), flush=True)
print(sys.argv[1] if len(sys.argv) > 1 else "", "resnet20 s/image", round(float(np.median(ts)), 4), [round(v, 4) for v in ts])
