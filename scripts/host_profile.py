"""cProfile of one encrypted ResNet-20 inference's host side (N=2^16, depth 12):
where the host enqueue time goes (Python vs the C-ABI calls)."""
import cProfile
import pstats
import sys

sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M


def norm(x):
    return (x - 0.5) / 0.2887


spec = M.calibrate_relu_scales(M.resnet20(ring=65536, depth_budget=int(sys.argv[1]) if len(sys.argv) > 1 else 12),
                               [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)])
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
em = M.EncryptedModel(spec)
for _ in range(3):
    em.infer(x)
pr = cProfile.Profile()
pr.enable()
em.infer(x)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
