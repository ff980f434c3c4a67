"""VGG-16 s/image after the bench's headline section (torch CUDA init, a key-sharing clone
driven from two threads) -- diagnostic for the bench-only slowdown."""
import sys
import threading

sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

sys.argv = sys.argv[:1]
import bench  # noqa: E402

torch.cuda.set_device(0)
step = int(__import__('os').environ.get("STEP", "3"))
if step >= 1:
    spec, x = bench.head_spec(11)
    em = M.EncryptedModel(spec)
    xin = em.encrypt_input(x)
    em.forward(xin)
    if step >= 2:
        tw = em.clone()
        x2 = tw.encrypt_input(x)
        th = [threading.Thread(target=lambda e, v: [e.forward(v) for _ in range(2)], args=a) for a in ((em, xin), (tw, x2))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        del tw, x2
    em.ctx.sync()
    del em, xin
    fh.api.release_memory()


def norm(v):
    return (v - 0.5) / 0.2887


spec = M.calibrate_relu_scales(M.vgg16_paper(ring=65536, depth_budget=11),
                               [norm(np.random.default_rng(5002 + i).uniform(0, 1, (3, 32, 32))) for i in range(4)])
x = norm(np.random.default_rng(5001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
for _ in range(3):
    em.infer(x)
print("step", step, [round(em.infer(x).wall_ms / 1e3, 4) for _ in range(3)], flush=True)
