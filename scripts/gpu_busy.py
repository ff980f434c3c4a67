"""GPU busy fraction (NVML utilization: share of time a kernel is running)
while encrypted ResNet-20 inferences run back to back; tells whether the
host enqueue or the device is the bottleneck."""
import sys
import threading
import time

sys.path.insert(0, '.')
import numpy as np
import pynvml
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


which = sys.argv[1] if len(sys.argv) > 1 else "resnet20"
if which == "resnet20":
    spec = M.resnet20(ring=65536, depth_budget=12)
    spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                          for i in range(6)])
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
else:
    spec = M.lenet5(ring=32768, depth_budget=12)
    x = np.random.default_rng(3001).uniform(0, 1, (1, 28, 28))
em = M.EncryptedModel(spec)
em.infer(x)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = [False]


def sampler():
    while not stop[0]:
        samples.append(pynvml.nvmlDeviceGetUtilizationRates(h).gpu)
        time.sleep(0.02)


th = threading.Thread(target=sampler)
th.start()
t0 = time.perf_counter()
n = 0
while time.perf_counter() - t0 < 8.0:
    em.infer(x)
    n += 1
stop[0] = True
th.join()
print(f"{which}: {n} inferences in {time.perf_counter() - t0:.2f}s; NVML utilization median {np.median(samples):.0f}% "
      f"mean {np.mean(samples):.1f}% over {len(samples)} samples")
