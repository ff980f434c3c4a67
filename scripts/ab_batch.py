"""ResNet-20 128-bit s/image: forward() one image at a time vs forward_batch() of B images in
lockstep (bootstraps through bootstrap_many), optionally F batch streams in flight
(key-sharing clones, one host thread each).  Usage: ab_batch.py [B ...]; env FLIGHT=F."""
import os
import sys
import threading
import time

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.resnet20(ring=65536, depth_budget=11)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                      for i in range(3)])
em = M.EncryptedModel(spec)
REPS = int(os.environ.get("REPS", "4"))
if os.environ.get("SWITCH"):
    sys.setswitchinterval(float(os.environ["SWITCH"]))
F = int(os.environ.get("FLIGHT", "1"))
em.batch_relu = os.environ.get("BATCH_RELU", "1") != "0"
ems = [em] + [em.clone() for _ in range(F - 1)]


def timed(fn, reps=REPS, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts))


def run_all(B):
    STEPS = int(os.environ.get("STEPS", "1"))  # forward passes per thread between synchronisations

    def work(e, vs):
        for _ in range(STEPS):
            if B == 0:
                e.forward(vs[0])
            else:
                e.forward_batch(vs)
        e.ctx.sync()
    ins = []
    for k, e in enumerate(ems):
        ins.append([e.encrypt_input(norm(np.random.default_rng(4001 + 10 * k + i).uniform(0, 1, (3, 32, 32))))
                    for i in range(max(B, 1))])

    def once():
        th = [threading.Thread(target=work, args=(e, vs)) for e, vs in zip(ems, ins)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    return timed(once) / (max(B, 1) * F * STEPS)


for B in [int(a) for a in sys.argv[1:]] or [0, 1, 2, 4]:
    try:
        print(f"B={B} (0 = forward) x {F} in flight: {run_all(B):.4f} s/image", flush=True)
        import torch
        free, total = torch.cuda.mem_get_info()
        print(f"   device memory free {free / 1e9:.1f} of {total / 1e9:.1f} GB", flush=True)
    except Exception as ex:  # noqa: BLE001
        print(f"B={B}: failed: {str(ex)[:200]}", flush=True)
