"""CPU: the slot-domain algebra of sparse-slot bootstrapping (csrc/bootstrap.cpp,
DESIGN.md section 3.1), restated in numpy on a small ring (N = 2^6, S = 32) and
checked end to end with the modular reduction done exactly:

  mask to [0, n) -> replicate (sum_j rot(x, j n)) -> "ModRaise" (+ integer I on
  every coefficient) -> trace (sum_j rot(., j n)) -> CtS (stages n..2, / g, then
  D = [1 | -i]) with offsets reduced mod n -> v + conj(v) -> EvalMod (exact frac
  of each real slot / 2) -> StC (P = [1 | i] + [i | 1] rot_n at period 2n, stages
  2..n at period n, output mask) == the input's first n slots, zeros after.

The matrices follow Bootstrapper::stage / mul / reduce_period line for line
(same twiddle indexing through rotgroup = 5^j mod 2N and the ksi table); the
full-slot pipeline (n = S, two EvalMod halves) is checked the same way.
"""
import numpy as np
import pytest

LOGN = 6
N = 1 << LOGN
S = N // 2
M = 2 * N
ROT = [pow(5, j, M) for j in range(S)]
KSI = np.exp(2j * np.pi * np.arange(M + 1) / M)


def decode(t):
    """slots of a real coefficient vector: z_j = sum_k t_k zeta^{k 5^j}"""
    k = np.arange(N)
    return np.array([np.sum(t * KSI[(k * ROT[j]) % M]) for j in range(S)])


def encode(z):
    A = np.array([[KSI[(k * ROT[j]) % M] for k in range(N)] for j in range(S)])
    return np.linalg.solve(np.vstack([A, A.conj()]), np.concatenate([z, z.conj()])).real


def signed_off(d, period=S):
    d %= period
    return d - period if d > period // 2 else d


def stage(length, inverse):
    """Bootstrapper::stage: one special-FFT stage as a 3-diagonal slot matrix"""
    lenh, lenq = length // 2, 4 * length
    d0, dp, dm = (np.zeros(S, complex) for _ in range(3))
    for k in range(S):
        p = k % length
        j = p if p < lenh else p - lenh
        idx = ((ROT[j] % lenq) if not inverse else (lenq - ROT[j] % lenq)) * (M // lenq)
        w = KSI[idx]
        if not inverse:
            if p < lenh:
                d0[k], dp[k] = 1, w
            else:
                d0[k], dm[k] = -w, 1
        elif p < lenh:
            d0[k], dp[k] = .5, .5
        else:
            d0[k], dm[k] = -.5 * w, .5 * w
    m = {}
    for off, d in ((0, d0), (signed_off(lenh), dp), (signed_off(-lenh), dm)):
        m[off] = m.get(off, np.zeros(S, complex)) + d
    return m


def mul(A, B):
    """(A B) x = sum_{a,b} (A_a (*) rot(B_b, a)) (*) rot(x, a + b)"""
    out = {}
    for a, da in A.items():
        for b, db in B.items():
            o = signed_off(a + b)
            out[o] = out.get(o, np.zeros(S, complex)) + da * np.roll(db, -a)
    return {k: v for k, v in out.items() if np.abs(v).max() > 1e-300}


def reduce_period(m, period):
    if period >= S:
        return m
    out = {}
    for d, v in m.items():
        r = signed_off(d, period)
        out[r] = out.get(r, np.zeros(S, complex)) + v
    return out


def apply(m, x):
    return sum(d * np.roll(x, -off) for off, d in m.items())


def rot(v, d):
    return np.roll(v, -d)


def pipeline(n, rng):
    g = S // n
    m = np.zeros(S, complex)
    m[:n] = rng.uniform(-1, 1, n) * 1e-3 + 1j * rng.uniform(-1, 1, n) * 1e-3
    garbage = rng.uniform(-1, 1, S) * 1e-3
    x_slots = m + np.where(np.arange(S) >= n, garbage, 0)  # inactive slots carry garbage
    # mask + replicate (one limb)
    xm = x_slots * (np.arange(S) < n)
    xr = sum(rot(xm, j * n) for j in range(g))
    # ModRaise: + integer overflow polynomial
    t = encode(xr) + rng.integers(-12, 13, N)
    y = decode(t)
    y = sum(rot(y, j * n) for j in range(g))  # trace
    cts = []
    length = n
    while length >= 2:
        cts.append(stage(length, True))
        length //= 2
    A = cts[0]
    for st in cts[1:]:
        A = mul(st, A)
    A = {k: v / g for k, v in A.items()}
    if n < S:
        dv = np.array([1 if (k % (2 * n)) < n else -1j for k in range(S)])
        A = mul({0: dv}, A)
        A = reduce_period(A, n)
    v = apply(A, y)
    if n < S:
        w = (v + v.conj())
        assert np.abs(w.imag).max() < 1e-9  # one REAL ciphertext holds all 2n coefficients
        wf = w.real / 2 - np.round(w.real / 2)  # exact EvalMod
        da = np.array([1 if (k % (2 * n)) < n else 1j for k in range(S)])
        db = np.array([1j if (k % (2 * n)) < n else 1 for k in range(S)])
        B1 = {0: da.astype(complex), signed_off(n): db.astype(complex)}
        length = 2
        while length < n:
            B1 = mul(stage(length, False), B1)
            length *= 2
        B2 = mul({0: (np.arange(S) < n).astype(complex)}, stage(n, False))
        out = apply(reduce_period(B2, n), apply(reduce_period(B1, 2 * n), wf))
    else:
        ys0 = (v + v.conj()).real
        ys1 = (1j * (v.conj() - v)).real
        z = (ys0 / 2 - np.round(ys0 / 2)) + 1j * (ys1 / 2 - np.round(ys1 / 2))
        B = stage(2, False)
        length = 4
        while length <= S:
            B = mul(stage(length, False), B)
            length *= 2
        out = apply(B, z)
    return m, out


@pytest.mark.parametrize("n", [S, S // 2, S // 4, S // 8])
def test_sparse_slot_bootstrap_algebra(n):
    m, out = pipeline(n, np.random.default_rng(n))
    assert np.abs(out[:n] - m[:n]).max() < 1e-12
    if n < S:
        assert np.abs(out[n:]).max() < 1e-12
