"""ModRaise -> CoeffsToSlots noise inside a real bootstrap at N = 2^16 (dense
secret via the sparse-secret encapsulation vs sparse main secret), with the
canonical-embedding inverse computed by a length-2N FFT (diagnostic)."""
import dataclasses
import sys

sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import api, model as M

N = 65536
S = N // 2
M2 = 2 * N
g = np.array([pow(5, j, M2) for j in range(S)], dtype=np.int64)


def coeffs_of_slots(z):
    """real coefficients c (N) with slots z_j = sum_k c_k zeta^{k g_j}, zeta = e^{i pi / N}"""
    Z = np.zeros(M2, complex)
    Z[g] = z
    Z[(M2 - g) % M2] = np.conj(z)
    # c_k = (1/N) sum_{t odd} Z[t] zeta^{-k t}
    c = np.fft.fft(Z)[:N] / N  # sum_t Z[t] e^{-2 pi i k t / 2N}
    return c.real


brv = np.array([int(format(i, "015b")[::-1], 2) for i in range(S)])
spec = M.resnet20(ring=65536, depth_budget=12)
base = M.ckks_config(spec, True, security=0)
rng = np.random.default_rng(5)
v = rng.uniform(-1, 1, S)
for name, cfg in {"sparse": base, "dense": dataclasses.replace(base, hamming_weight=0)}.items():
    ctx = fh.SlotContext(cfg)
    q0 = float(ctx.primes[0])
    x0 = fh.level_down(fh.SlotVector.encode(ctx, v), 1)
    m = coeffs_of_slots(x0.slots() * x0.scale())  # message coefficients (incl. noise)
    r4 = api.bootstrap_stage(x0, 4)
    t = coeffs_of_slots(r4.slots_complex() * r4.scale()) / q0
    I = np.round(t - m / q0)
    res = (t - m / q0 - I) * q0
    print(name, "ModRaise: max|I|", np.abs(I).max(), "residual (coeff units)", np.abs(res).max(), flush=True)
    r1 = api.bootstrap_stage(r4, 1).slots_complex()
    tc = t[:S] + 1j * t[S:]
    want = tc[brv] / 34.0
    print(name, "CtS: max err", np.abs(r1 - want).max(), "magnitude", np.abs(want).max(),
          "err in m/q0 units x107x5215:", np.abs(r1 - want).max() * 34 * 107 * 5215 / 34, flush=True)
    y = fh.bootstrap(x0)
    print(name, "bootstrap err", np.abs(y.slots() - x0.slots()).max(), flush=True)
    del ctx
