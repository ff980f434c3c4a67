"""VGG-16 s/image alone vs after another model in the same process (diagnostic)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


def vgg_time(tag):
    spec = M.calibrate_relu_scales(M.vgg16_paper(ring=65536, depth_budget=11),
                                   [norm(np.random.default_rng(5002 + i).uniform(0, 1, (3, 32, 32))) for i in range(4)])
    x = norm(np.random.default_rng(5001).uniform(0, 1, (3, 32, 32)))
    fh.api.release_memory()
    em = M.EncryptedModel(spec)
    for _ in range(3):
        em.infer(x)
    ts = [em.infer(x).wall_ms / 1e3 for _ in range(3)]
    print(tag, [round(t, 4) for t in ts], "keys GB", round(em.ctx.key_bytes() / 1e9, 1), flush=True)
    del em


vgg_time("first")
if len(sys.argv) > 1:
    spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=25),
                                   [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)])
    em = M.EncryptedModel(spec, security=0)
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
    for _ in range(3):
        em.infer(x)
    del em
vgg_time("second")
