"""Throughput of R concurrent ResNet-20 inferences (R independent engine contexts,
one CUDA stream each, one host thread each) vs one at a time (diagnostic)."""
import sys
import threading
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=11),
                               [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
ems = [M.EncryptedModel(spec)]
ems += [ems[0].clone() for _ in range(R - 1)]  # key-sharing clones
xins = [em.encrypt_input(x) for em in ems]
for em, xi in zip(ems, xins):
    em.forward(xi)
    em.forward(xi)
    em.ctx.sync()
# one at a time
t0 = time.perf_counter()
for _ in range(K):
    o = ems[0].forward(xins[0])
ems[0].ctx.sync()
single = (time.perf_counter() - t0) / K


def run(i):
    for _ in range(K):
        ems[i].forward(xins[i])
    ems[i].ctx.sync()


th = [threading.Thread(target=run, args=(i,)) for i in range(R)]
t0 = time.perf_counter()
for t in th:
    t.start()
for t in th:
    t.join()
conc = (time.perf_counter() - t0) / (K * R)
print(f"R={R}: single {single:.4f} s/image, concurrent {conc:.4f} s/image ({single / conc:.2f}x), "
      f"keys {sum(e.ctx.key_bytes() for e in ems) / 1e9:.1f} GB", flush=True)
