"""Kernel-level breakdown of one ResNet-20 building block at N=2^16 (depth 12,
29 limbs, bootstrapping chain).  Run under
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ...
the profiled region (cudaProfilerStart/Stop) holds exactly one call of the
chosen block after a warm-up call.  Blocks: conv2 (unit2_1 2x2/s2 16->32 on
32x32), conv3 (64->64 3x3 on 8x8), relu, bootstrap."""
import ctypes
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M

which = sys.argv[1] if len(sys.argv) > 1 else "conv2"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 12
spec = M.resnet20(ring=65536, depth_budget=depth)
ctx = fh.SlotContext(M.ckks_config(spec, True, security=int(__import__('os').environ.get('FHEON_SECURITY', '0'))))
rng = np.random.default_rng(5)
cudart = ctypes.CDLL("libcudart.so.12")


def block():
    if which == "conv2":
        C, W, F = 16, 32, 32
        x = fh.SlotVector.encode(ctx, rng.uniform(-1, 1, C * W * W))
        w = rng.normal(0, 0.2, (F, C, 2, 2))
        return lambda: fh.convolution(fh.PackedTensor(x, C, W), fh.ConvConfig(C, F, 2, 2, 0),
                                      fh.KernelTensor(w)).data
    if which == "conv3":
        C, W, F = 64, 8, 64
        x = fh.SlotVector.encode(ctx, rng.uniform(-1, 1, C * W * W))
        w = rng.normal(0, 0.05, (F, C, 3, 3))
        return lambda: fh.convolution(fh.PackedTensor(x, C, W),
                                      fh.ConvConfig(C, F, 3, 1, 1, fh.ConvMode.special3x3), fh.KernelTensor(w)).data
    if which == "relu":
        x = fh.SlotVector.encode(ctx, rng.uniform(-1, 1, 4096))
        return lambda: fh.secure_relu(x, fh.ReluConfig(8.0, 59, 4096))
    if which == "bootstrap":
        x = fh.level_down(fh.SlotVector.encode(ctx, rng.uniform(-1, 1, 32768)), 1)
        return lambda: fh.bootstrap(x)
    raise SystemExit(f"unknown block {which}")


fn = block()
fn()
ctx.sync()
ctx.reset_stats()
cudart.cudaProfilerStart()
out = fn()
ctx.sync()
cudart.cudaProfilerStop()
print(which, ctx.stats(), "level", out.level())
