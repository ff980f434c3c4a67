"""One encrypted ResNet-20 inference inside a cudaProfilerStart/Stop range (for
ncu --profile-from-start off launch lists)."""
import ctypes
import sys

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


depth = int(sys.argv[1]) if len(sys.argv) > 1 else 12
spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=depth),
                               [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
for _ in range(3):
    em.infer(x)
cudart = ctypes.CDLL("libcudart.so.12")
cudart.cudaProfilerStart()
r = em.infer(x)
em.ctx.sync()
cudart.cudaProfilerStop()
print("launches", r.stats["launches"])
