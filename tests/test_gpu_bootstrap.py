"""GPU: CKKS bootstrapping, the realisation of the reference's bootstrap()
(proj/src/backend.cpp:233-249: slot values preserved, level := depth budget,
one `bootstrap` trace event).  Each stage is checked against an independent
numpy model of the canonical embedding U (z_j = sum_k w_k zeta^{5^j k}):
CoeffsToSlots = B U^{-1} / (2 (K+1)), EvalMod = sin(2 pi (K+1) u),
SlotsToCoeffs = U B q0 / (2 pi Delta_0), ModRaise = m + q0 I with integer I.
"""
import numpy as np
import pytest

import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import api

pytestmark = pytest.mark.gpu

LOGN, L = 12, 24
N, S = 1 << LOGN, 1 << (LOGN - 1)


@pytest.fixture(scope="module", params=["sparse", "sse"])
def bctx(request):
    """sparse: the main secret itself sparse (h = 64); sse: a uniform ternary main
    secret, bootstrapping through the sparse-secret encapsulation (level-0 switch
    to an ephemeral h = 64 secret, ModRaise, switch back)."""
    cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=L, special_limbs=8, special_bits=60,
                           seed=5, hamming_weight=64 if request.param == "sparse" else 0, bootstrap=True,
                           boot_scale_bits=55, allow_insecure=True)
    ctx = fh.SlotContext(cfg)
    M = 2 * N
    rot = np.array([pow(5, j, M) for j in range(S)], dtype=np.int64)
    U = np.exp(2j * np.pi * ((rot[:, None] * np.arange(S)[None, :]) % M) / M)
    brv = np.array([int(format(i, f"0{LOGN - 1}b")[::-1], 2) for i in range(S)])
    return ctx, U, brv


def test_depth_budget_and_chain(bctx):
    ctx, _, _ = bctx
    info = api.bootstrap_info(ctx)
    assert info["depth"] == 3 + 7 + 3 + 3
    assert ctx.depth_budget() == L - 1 - info["depth"]
    T = np.log2(ctx.scales)
    assert abs(T[0] - 40) < 0.01 and abs(T[-1] - 55) < 0.01


def test_coeffs_to_slots_stage(bctx):
    ctx, U, brv = bctx
    rng = np.random.default_rng(0)
    q0 = float(ctx.primes[0])
    z = rng.uniform(-1, 1, S) * q0 / ctx.scales[-1]  # reinterpreted slots of O(1)
    x = fh.SlotVector.encode_top(ctx, z)
    y = api.bootstrap_stage(x, 1).slots_complex()
    want = np.linalg.solve(U, z * x.scale() / q0)[brv] / (2 * 17.0)
    assert np.abs(y - want).max() < 1e-9 * max(1.0, np.abs(want).max())


def test_evalmod_stage(bctx):
    ctx, _, _ = bctx
    rng = np.random.default_rng(1)
    u = rng.uniform(-0.95, 0.95, S)
    x = fh.level_down(fh.SlotVector.encode_top(ctx, u), L - 3)
    e = api.bootstrap_stage(x, 2).slots()
    assert np.abs(e - np.sin(2 * np.pi * 17.0 * u)).max() < 1e-5


def test_slots_to_coeffs_stage(bctx):
    ctx, U, brv = bctx
    rng = np.random.default_rng(2)
    w = rng.uniform(-1, 1, S) * 1e-3
    x = fh.SlotVector.encode_top(ctx, w)
    s = api.bootstrap_stage(x, 3).slots_complex()
    want = (U @ w[brv]) * float(ctx.primes[0]) / (2 * np.pi * ctx.scales[0])
    assert np.abs(s - want).max() < 1e-6 * max(1.0, np.abs(want).max())


def test_modraise_integer_overflow(bctx):
    ctx, U, _ = bctx
    rng = np.random.default_rng(3)
    z = rng.uniform(-1, 1, S)
    x0 = fh.level_down(fh.SlotVector.encode(ctx, z), 1)
    r = api.bootstrap_stage(x0, 4)
    assert r.limbs() == L
    t = np.linalg.solve(U, r.slots_complex())          # (m + q0 I) / q0 in complex packing
    m = np.linalg.solve(U, z * ctx.scales[0] / float(ctx.primes[0]))
    I = t - m
    assert np.abs(I - np.round(I)).max() < 1e-6       # integer overflow polynomial
    assert np.abs(np.round(I)).max() <= 16            # within the EvalMod range K


@pytest.mark.parametrize("mag", [1.0, 8.0])
def test_bootstrap_identity_level_and_trace(bctx, mag):
    ctx, _, _ = bctx
    rng = np.random.default_rng(int(mag))
    v = rng.uniform(-mag, mag, S)
    x = fh.level_down(fh.SlotVector.encode(ctx, v), 1)
    rec = ctx.attach_recorder()
    y = fh.bootstrap(x)
    ev = [(e.kind, e.value) for e in rec.snapshot()]
    ctx.detach_recorder()
    assert y.level() == ctx.depth_budget()
    assert ev == [("bootstrap", ctx.depth_budget())]
    assert np.abs(y.slots() - v).max() < 1e-4
    # refreshed ciphertexts compute again
    z = fh.mult_plain(y, np.full(S, 0.5))
    assert np.abs(z.slots() - 0.5 * v).max() < 1e-4


def test_bootstrap_from_higher_level(bctx):
    ctx, _, _ = bctx
    rng = np.random.default_rng(9)
    v = rng.uniform(-1, 1, S)
    y = fh.bootstrap(fh.SlotVector.encode(ctx, v))
    assert y.level() == ctx.depth_budget()
    assert np.abs(y.slots() - v).max() < 1e-4


def test_bootstrap_requires_enabled_context():
    cfg = fh.ContextConfig(4096, 2048, 5, fh.CryptoMetadata(50, 40, 3), limbs=6, special_limbs=2,
                           allow_insecure=True)
    ctx = fh.SlotContext(cfg)
    x = fh.SlotVector.encode(ctx, [1.0])
    with pytest.raises(fh.NotImplementedInEngine):
        fh.bootstrap(x)


def test_sse_keys_and_switches_bit_exact():
    """Sparse-secret encapsulation keys (ids 2: s -> s_b on q_0 and P only, 4:
    s_b -> s) and the two key switches of ModRaise, bit-exact against the
    oracle's restatement (ock_set_boot_secret / ock_keygen)."""
    from oracle.ckks_oracle import Oracle
    cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=L, special_limbs=8, special_bits=60,
                           seed=6, bootstrap=True, boot_scale_bits=55, allow_insecure=True)
    ctx = fh.SlotContext(cfg)
    orc = Oracle.from_chain(LOGN, ctx.primes, ctx.scales, L, 8, 3, seed=6)
    orc.set_boot_secret(64)
    k2, k4 = orc.keygen(2), orc.keygen(4)
    assert np.array_equal(ctx.download_key(2), k2)
    assert np.array_equal(ctx.download_key(4), k4)
    assert not k2[0, :, 1:L].any() and not k2[1:].any()  # the sparse sample lives on q_0 and P only
    rng = np.random.default_rng(8)
    ct = orc.encrypt(rng.uniform(-1, 1, S), 3)
    x1 = fh.SlotVector.from_words(ctx, np.ascontiguousarray(ct[:, :1]), float(orc.T[0]))
    ks = fh.keyswitch_raw(x1, 2, 1).words()
    k0, k1 = orc.keyswitch(np.ascontiguousarray(ct[1, :1]), k2, 1)
    assert np.array_equal(ks[0], k0) and np.array_equal(ks[1], k1)
    xt = fh.SlotVector.from_words(ctx, ct, float(orc.T[-1]))
    ks = fh.keyswitch_raw(xt, 4, 1).words()
    k0, k1 = orc.keyswitch(ct[1], k4, 1)
    assert np.array_equal(ks[0], k0) and np.array_equal(ks[1], k1)


@pytest.fixture(scope="module", params=["sparse", "sse"])
def sctx(request):
    """Contexts with the sparse-slot variants (n = S/2, S/4, S/8)."""
    cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=L, special_limbs=8, special_bits=60,
                           seed=7, hamming_weight=64 if request.param == "sparse" else 0, bootstrap=True,
                           boot_scale_bits=55, allow_insecure=True, boot_sparse=3)
    return fh.SlotContext(cfg)


@pytest.mark.parametrize("active", [S // 2, 700, S // 8, 3, S // 2 + 1])
def test_bootstrap_active_sparse_slots(sctx, active):
    """bootstrap(v, active): the smallest sparse-slot variant n >= active keeps
    slots [0, n) (the input's), zeroes [n, S), lands on the depth budget with one
    bootstrap trace event -- the reference's bootstrap() on the slots that matter."""
    n = S
    for k in (1, 2, 3):
        if active <= S >> k:
            n = S >> k
    rng = np.random.default_rng(active)
    v = rng.uniform(-1, 1, S)
    x = fh.level_down(fh.SlotVector.encode(sctx, v), 2)  # level 1
    rec = sctx.attach_recorder()
    y = fh.bootstrap(x, active)
    ev = [(e.kind, e.value) for e in rec.snapshot()]
    sctx.detach_recorder()
    assert y.level() == sctx.depth_budget()
    assert ev == [("bootstrap", sctx.depth_budget())]
    out = y.slots()
    assert np.abs(out[:n] - v[:n]).max() < 1e-4
    if n < S:
        assert np.abs(out[n:]).max() < 1e-4
    else:
        assert np.abs(out - v).max() < 1e-4
    # refreshed ciphertexts compute again
    z = fh.mult_plain(y, np.full(S, 0.5))
    assert np.abs(z.slots()[:active] - 0.5 * v[:active]).max() < 1e-4


def test_bootstrap_active_level0_runs_full(sctx):
    """At level 0 there is no level for the mask: the full pipeline runs."""
    rng = np.random.default_rng(11)
    v = rng.uniform(-1, 1, S)
    x = fh.level_down(fh.SlotVector.encode(sctx, v), 1)  # level 0
    y = fh.bootstrap(x, 100)
    assert np.abs(y.slots() - v).max() < 1e-4
    with pytest.raises(fh.ShapeError):
        fh.bootstrap(x, S + 1)


@pytest.mark.parametrize("active,clean,level", [(S // 4, False, 2), (S // 8, True, 1), (S // 2, False, 3)])
def test_bootstrap_many_bit_identical(sctx, active, clean, level):
    """bootstrap_many (the images of a batched inference in lockstep: keys and
    diagonals read once per batch) returns, per input, the very words of
    bootstrap(x, active, clean) -- and one bootstrap trace event per input."""
    rng = np.random.default_rng(100 + active)
    vs = [rng.uniform(-1, 1, S) for _ in range(3)]
    if clean:
        for v in vs:
            v[active:] = 0.0
    xs = [fh.level_down(fh.SlotVector.encode(sctx, v), level) for v in vs]
    singles = [fh.bootstrap(x, active, clean=clean) for x in xs]
    rec = sctx.attach_recorder()
    many = fh.bootstrap_many(xs, active, clean=clean)
    ev = [(e.kind, e.value) for e in rec.snapshot()]
    sctx.detach_recorder()
    assert ev == [("bootstrap", sctx.depth_budget())] * 3
    for s, m, v in zip(singles, many, vs):
        assert m.level() == s.level() == sctx.depth_budget()
        assert np.array_equal(m.words(), s.words())
        assert np.abs(m.slots()[:active] - v[:active]).max() < 1e-4


def test_bootstrap_many_mixed_levels_and_full(sctx):
    """Inputs on different levels (or no sparse variant: level 0 without `clean`)
    run one after the other with the same results."""
    rng = np.random.default_rng(77)
    vs = [rng.uniform(-1, 1, S) for _ in range(2)]
    xs = [fh.level_down(fh.SlotVector.encode(sctx, vs[0]), 2), fh.level_down(fh.SlotVector.encode(sctx, vs[1]), 3)]
    many = fh.bootstrap_many(xs, S // 4)
    for x, m in zip(xs, many):
        assert np.array_equal(m.words(), fh.bootstrap(x, S // 4).words())
    x0 = [fh.level_down(fh.SlotVector.encode(sctx, v), 1) for v in vs]  # level 0: full pipeline
    for m, v in zip(fh.bootstrap_many(x0, 100), vs):
        assert np.abs(m.slots() - v).max() < 1e-4
    assert fh.bootstrap_many([], 10) == []
