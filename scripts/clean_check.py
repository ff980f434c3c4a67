"""Which layer outputs are exactly zero beyond the tensor's active slots?
(ResNet-20 128-bit, layer by layer, max |slot| past C*W*W after every layer.)"""
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.resnet20(ring=65536, depth_budget=11)
spec = M.calibrate_relu_scales(spec, [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32)))
                                      for i in range(3)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
v = fh.SlotVector.encode(em.ctx, x.reshape(-1))


def walk(layers, v, ind=0):
    for b in layers:
        if b.type == "residual":
            body = walk(b.body, v, ind + 2)
            skip = walk(b.downsample, v, ind + 2) if b.downsample else v
            out = fh.add(body, skip)
        else:
            out = em._run(b, v, None)
        packed, C, W, n = b.out_shape
        act = C * W * W if packed else n
        s = out.slots()
        print(" " * ind, f"{b.type:16s} {b.name:22s} level {out.level():2d} active {act:6d} max|beyond| {np.abs(s[act:]).max():.2e} max|active| {np.abs(s[:act]).max():.2e}", flush=True)
        v = out
    return v


walk(em.layers, v)
