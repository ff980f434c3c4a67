"""Does a preceding model context slow ResNet-20 (depth 25)?  Times ResNet-20
alone, then after LeNet-5 contexts were built and dropped (the bench order)."""
import gc
import subprocess
import sys
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


def clocks():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,memory.used",
                           "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()


cal = [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)]
xr = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=25), cal)


def run_resnet(tag):
    em = M.EncryptedModel(spec)
    em.infer(xr)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        em.infer(xr)
        ts.append(time.perf_counter() - t0)
    print(tag, [round(t, 3) for t in ts], clocks(), flush=True)
    del em
    gc.collect()


if sys.argv[1:] == ["after"]:
    xl = np.random.default_rng(3001).uniform(0, 1, (1, 28, 28))
    for d in (25, 12):
        em = M.EncryptedModel(M.lenet5(ring=32768, depth_budget=d))
        em.infer(xl)
        em.infer(xl)
        del em
        gc.collect()
    print("after lenet:", clocks(), flush=True)
run_resnet("resnet20 d25")
run_resnet("resnet20 d25 again")
