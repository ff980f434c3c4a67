import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import api
logN, L = 12, 24
N = 1 << logN; S = N // 2
cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=L, special_limbs=6, special_bits=60,
                       seed=5, hamming_weight=64, bootstrap=True)
ctx = fh.SlotContext(cfg)
info = api.bootstrap_info(ctx)
print("depth", info["depth"], "budget", ctx.depth_budget(), "cos deg", len(info["cos_coeffs"]) - 1, flush=True)
q0 = float(ctx.primes[0]); T = ctx.scales
K1 = 17.0
# numpy model of U (decode matrix): z_j = sum_k w_k zeta^{5^j k}, k < S
M = 2 * N
rot = np.array([pow(5, j, M) for j in range(S)], dtype=np.int64)
k = np.arange(S)
U = np.exp(2j * np.pi * ((rot[:, None] * k[None, :]) % M) / M)
brv = np.array([int(format(i, f"0{logN-1}b")[::-1], 2) for i in range(S)])
rng = np.random.default_rng(0)
z = rng.uniform(-1, 1, S)
# stage 1: CoeffsToSlots on a top-level ciphertext, scale reinterpreted as q0
x = fh.SlotVector.encode_top(ctx, z)
y = api.bootstrap_stage(x, 1).slots_complex()
zp = z * x.scale() / q0
w = np.linalg.solve(U, zp)
want = w[brv] / (2 * K1)
print("CtS err", np.abs(y - want).max(), "scale of want", np.abs(want).max(), flush=True)
# stage 2: EvalMod on u in [-1, 1]
u = rng.uniform(-1, 1, S) * 0.9
xu = fh.level_down(fh.SlotVector.encode_top(ctx, u), L - 3)
e = api.bootstrap_stage(xu, 2).slots()
print("EvalMod err", np.abs(e - np.sin(2 * np.pi * K1 * u)).max(), flush=True)
# stage 3: SlotsToCoeffs on w (real input)
wv = rng.uniform(-1, 1, S)
xw = fh.SlotVector.encode_top(ctx, wv)
s = api.bootstrap_stage(xw, 3).slots_complex()
want3 = (U @ wv) * q0 / (2 * np.pi * T[0])
print("StC err", np.abs(s - want3).max(), "mag", np.abs(want3).max(), flush=True)
# stage 4: ModRaise
x0 = fh.level_down(fh.SlotVector.encode(ctx, z), 1)
r = api.bootstrap_stage(x0, 4)
zr = r.slots_complex()  # = U(m + q0 I) / q0
I_est = np.linalg.solve(U, zr)
mt = np.linalg.solve(U, z * T[0] / q0)
print("ModRaise: I range", np.abs(np.round(I_est - mt)).max(), "frac err", np.abs((I_est - mt) - np.round(I_est - mt)).max(), flush=True)
