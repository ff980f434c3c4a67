"""Kernel-level breakdown of one whole encrypted inference (ResNet-20 at N=2^16
or LeNet-5 at N=2^15, the bench's model configs).  Run under
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ...
the profiled region (cudaProfilerStart/Stop) holds exactly one inference after
warm-up inferences (weights encoded, keys generated, pools grown)."""
import ctypes
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M

which = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cudart = ctypes.CDLL("libcudart.so.12")


def norm(x):
    return (x - 0.5) / 0.2887


if which == "resnet20":
    spec = M.resnet20(ring=65536, depth_budget=depth)
    spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                          for i in range(6)])
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
else:
    spec = M.lenet5(ring=32768, depth_budget=depth)
    x = np.random.default_rng(3001).uniform(0, 1, (1, 28, 28))
em = M.EncryptedModel(spec, security=int(__import__('os').environ.get('FHEON_SECURITY', '0')))
for _ in range(2):
    em.infer(x)
em.ctx.sync()
em.ctx.reset_stats()
t0 = time.perf_counter()
cudart.cudaProfilerStart()
r = em.infer(x)
em.ctx.sync()
cudart.cudaProfilerStop()
print(which, depth, f"{time.perf_counter() - t0:.3f} s", em.ctx.stats(), flush=True)
