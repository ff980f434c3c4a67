"""GPU parity at the model runtime's PRODUCTION chains, bit-exact against the
CPU oracle (oracle/ckks_oracle.c) built over the engine's own primes
(Oracle.from_chain).

ResNet-20 at BASELINE configs[3] runs on model.ckks_config(resnet20(ring=2^16,
depth_budget=25), bootstrapping=True): N = 2^16, L = 42 limbs (55-bit q0, 25
application primes of ~40 bits, 16 bootstrapping primes of ~55 bits), K = 12
special primes, dnum = 3 digits balanced by prime bit size (digit_split = 1),
sparse secret h = 64.  Its digits hold more than 12 limbs, so every key switch
runs the 16-input tensor-core basis conversions (bconv_tc.cu dispatch_tc:
k_bconv_tc<16, 0> for ModUp, k_bconv_tc<16, 1> for ModDown with K + 2 = 14
inputs and for the fused relinearise-rescale ModDown with K + 3 = 15 inputs).
The MODE-2 kernels (K >= 14: no room for the two finishing columns) are forced
with K = 14 and K = 15 on a small ring.
"""
import numpy as np
import pytest

import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M
from oracle.ckks_oracle import Oracle

pytestmark = pytest.mark.gpu


def _digits(primes, L, dnum):
    """Balanced digit sizes (params.cpp balanced_digits / ock_set_digit_split)."""
    bits = [float(np.log2(float(q))) for q in primes[:L]]
    cap = M.balanced_widest(bits, dnum)
    sizes, acc, size = [], 0.0, 0
    for b in bits:
        if size == 15 or acc + b > cap:
            sizes.append(size)
            acc, size = 0.0, 0
        acc += b
        size += 1
    sizes.append(size)
    return sizes


@pytest.fixture(scope="module")
def prod():
    cfg = M.ckks_config(M.resnet20(ring=65536, depth_budget=25), True, security=0)
    ctx = fh.SlotContext(cfg)
    L, K = cfg.limbs, cfg.special_limbs
    orc = Oracle.from_chain(16, ctx.primes, ctx.scales, L, K, cfg.crypto.key_switch_digits, seed=cfg.seed,
                            hamming_weight=cfg.hamming_weight, digit_split=cfg.digit_split)
    assert (orc.primes == ctx.primes).all()
    return ctx, orc, cfg


def _ct(orc, seed, counter):
    vals = np.random.default_rng(seed).uniform(-1, 1, orc.S)
    return vals, orc.encrypt(vals, counter)


def test_production_chain_shape(prod):
    """The chain really is the production one and really reaches the 16-input kernels."""
    ctx, orc, cfg = prod
    assert (orc.N, cfg.limbs, cfg.special_limbs, cfg.crypto.key_switch_digits) == (65536, 42, 12, 3)
    sizes = _digits(ctx.primes, cfg.limbs, 3)
    assert sum(sizes) == 42 and len(sizes) == 3
    assert max(sizes) > 12, f"digits {sizes} would not reach KINP = 16"


def test_keys_bit_exact(prod):
    ctx, orc, _ = prod
    g = orc.galois(1)
    ctx.keygen_rotations([1])
    assert np.array_equal(ctx.download_key(g), orc.keygen(g))
    assert np.array_equal(ctx.download_key(0), orc.keygen(0))


@pytest.mark.parametrize("limbs", [42, 29, 14, 3])
def test_rotation_bit_exact(prod, limbs):
    """Top of the chain (3 digits of 13-15 limbs: KINP=16 ModUp) and lower
    levels (fewer and partial digits)."""
    ctx, orc, _ = prod
    _, ct = _ct(orc, 7000 + limbs, 3)
    ct = np.ascontiguousarray(ct[:, :limbs])
    x = fh.SlotVector.from_words(ctx, ct, float(orc.T[limbs - 1]))
    for t in (1, -3):
        got = fh.rotate(x, t).words()
        assert np.array_equal(got, orc.rotate(ct, t, orc.rotation_key(t))), f"t={t} limbs={limbs}"


def test_hoisted_and_batched_rotations_bit_exact(prod):
    ctx, orc, _ = prod
    _, ct = _ct(orc, 7100, 4)
    _, ct2 = _ct(orc, 7101, 5)
    x = fh.SlotVector.from_words(ctx, ct, float(orc.T[-1]))
    x2 = fh.SlotVector.from_words(ctx, ct2, float(orc.T[-1]))
    ts = [2, 17, -1000]
    keys = {t: orc.rotation_key(t) for t in ts}
    for t, y in zip(ts, fh.rotate_hoisted(x, ts)):
        assert np.array_equal(y.words(), orc.rotate(ct, t, keys[t]))
    ys = fh.rotate_many([x, x2, x2], [2, 2, 17])
    assert np.array_equal(ys[0].words(), orc.rotate(ct, 2, keys[2]))
    assert np.array_equal(ys[1].words(), orc.rotate(ct2, 2, keys[2]))
    assert np.array_equal(ys[2].words(), orc.rotate(ct2, 17, keys[17]))


@pytest.mark.parametrize("limbs", [42, 20])
def test_rotate_sum_bit_exact(prod, limbs):
    """Rotate-and-sum: every term's inner product in one Q+P accumulator, one
    16-input ModDown (ock_rotate_sum)."""
    ctx, orc, _ = prod
    cts = [np.ascontiguousarray(_ct(orc, 7200 + i, 6 + i)[1][:, :limbs]) for i in range(3)]
    ts = [1, 5, -7]
    xs = [fh.SlotVector.from_words(ctx, c, float(orc.T[limbs - 1])) for c in cts]
    y = fh.rotate_sum(xs, ts)
    want = orc.rotate_sum(cts, ts, [orc.rotation_key(t) for t in ts])
    assert np.array_equal(y.words(), want)
    # several groups, one sharing its key list (k_ks_inner_shared) and one not (k_ks_inner_sum)
    outs = fh.rotate_sum_many([[(xs[0], 1), (xs[0], 5)], [(xs[1], 1), (xs[2], -7)]])
    assert np.array_equal(outs[0].words(), orc.rotate_sum([cts[0]] * 2, [1, 5],
                                                          [orc.rotation_key(1), orc.rotation_key(5)]))
    assert np.array_equal(outs[1].words(), orc.rotate_sum([cts[1], cts[2]], [1, -7],
                                                          [orc.rotation_key(1), orc.rotation_key(-7)]))


@pytest.mark.parametrize("limbs", [42, 27, 9])
def test_mult_cipher_bit_exact(prod, limbs):
    """Tensor + relinearisation + rescale in ONE fused ModDown over K + 1 = 13
    special limbs (k_bconv_tc<16, 1>, ock_mult_cipher)."""
    ctx, orc, _ = prod
    a = np.ascontiguousarray(_ct(orc, 7300 + limbs, 9)[1][:, :limbs])
    b = np.ascontiguousarray(_ct(orc, 7400 + limbs, 10)[1][:, :limbs])
    sc = float(orc.T[limbs - 1])
    got = fh.mult_cipher(fh.SlotVector.from_words(ctx, a, sc), fh.SlotVector.from_words(ctx, b, sc))
    assert np.array_equal(got.words(), orc.mult_cipher(a, b, orc.relin_key()))


@pytest.mark.parametrize("limbs", [42, 16])
def test_keyswitch_and_rescale_bit_exact(prod, limbs):
    """Plain key switch (ModUp + inner product + plain ModDown, K + 2 = 14
    inputs) and rescale at the production chain."""
    ctx, orc, _ = prod
    ct = np.ascontiguousarray(_ct(orc, 7500 + limbs, 11)[1][:, :limbs])
    x = fh.SlotVector.from_words(ctx, ct, float(orc.T[limbs - 1]))
    g = orc.galois(1)
    ctx.keygen_rotations([1])
    ks = fh.keyswitch_raw(x, g, 1).words()
    k0, k1 = orc.keyswitch(ct[1], orc.keygen(g), 1)
    assert np.array_equal(ks[0], k0) and np.array_equal(ks[1], k1)
    assert np.array_equal(fh.rescale(x).words(), orc.rescale(ct))


@pytest.mark.parametrize("K", [14, 15])
def test_mode2_bconv_bit_exact(K):
    """K >= 14: the fused relinearise-rescale ModDown has K + 1 + 2 > 16 columns
    (MODE 2: finish on the CUDA cores); K = 15 also sends the plain ModDown
    (K + 2 > 16) there.  Rotation, key switch and mult_cipher bit-exact."""
    logN, L, dnum = 12, 20, 2
    cfg = fh.ContextConfig(1 << logN, 1 << (logN - 1), L - 1, fh.CryptoMetadata(50, 40, dnum), limbs=L,
                           special_limbs=K, special_bits=60, seed=31, allow_insecure=True)
    ctx = fh.SlotContext(cfg)
    orc = Oracle(logN, L, K, dnum, 50, 40, 60, 31)
    assert (orc.primes == ctx.primes).all()
    _, ct = _ct(orc, 7600 + K, 12)
    _, ct2 = _ct(orc, 7700 + K, 13)
    x = fh.SlotVector.from_words(ctx, ct, float(orc.T[-1]))
    y = fh.SlotVector.from_words(ctx, ct2, float(orc.T[-1]))
    assert np.array_equal(fh.rotate(x, 3).words(), orc.rotate(ct, 3, orc.rotation_key(3)))
    assert np.array_equal(fh.mult_cipher(x, y).words(), orc.mult_cipher(ct, ct2, orc.relin_key()))
    for limbs in (13, 4):
        c = np.ascontiguousarray(ct[:, :limbs])
        c2 = np.ascontiguousarray(ct2[:, :limbs])
        xs = fh.SlotVector.from_words(ctx, c, float(orc.T[limbs - 1]))
        ys = fh.SlotVector.from_words(ctx, c2, float(orc.T[limbs - 1]))
        assert np.array_equal(fh.mult_cipher(xs, ys).words(), orc.mult_cipher(c, c2, orc.relin_key()))
        assert np.array_equal(fh.rotate(xs, -5).words(), orc.rotate(c, -5, orc.rotation_key(-5)))


# ---- a 128-bit chain: ResNet-20 at depth budget 12, N = 2^16, uniform ternary
# secret, sparse-secret encapsulation (h_b = 32, EvalMod range 12) for bootstrapping,
# 60-bit CoeffsToSlots / EvalMod levels, L = 28, K = 5, dnum = 6 (log2 QP <= 1747,
# model.ckks_config security=128)

@pytest.fixture(scope="module")
def secure():
    cfg = M.ckks_config(M.resnet20(ring=65536, depth_budget=12), True)
    ctx = fh.SlotContext(cfg)
    sec = ctx.security()
    assert sec["meets_128"] and sec["log2_qp"] <= 1747 and cfg.hamming_weight == 0
    L, K = cfg.limbs, cfg.special_limbs
    orc = Oracle.from_chain(16, ctx.primes, ctx.scales, L, K, cfg.crypto.key_switch_digits, seed=cfg.seed,
                            digit_split=cfg.digit_split)
    orc.set_boot_secret(cfg.boot_hamming_weight or 64)
    return ctx, orc, cfg


def test_secure_chain_shape(secure):
    ctx, orc, cfg = secure
    dnum = cfg.crypto.key_switch_digits
    assert cfg.limbs == 12 + 1 + 15 and dnum > 3  # 15 bootstrapping levels (EvalMod range 12)
    assert len(_digits(ctx.primes, cfg.limbs, dnum)) == dnum
    assert max(int(q).bit_length() for q in ctx.primes) == 61  # 60-bit-target bootstrapping primes


@pytest.mark.parametrize("limbs", [28, 13, 1])
def test_secure_rotation_and_mult_cipher_bit_exact(secure, limbs):
    ctx, orc, _ = secure
    a = np.ascontiguousarray(_ct(orc, 7800 + limbs, 20)[1][:, :limbs])
    b = np.ascontiguousarray(_ct(orc, 7900 + limbs, 21)[1][:, :limbs])
    sc = float(orc.T[limbs - 1])
    x, y = fh.SlotVector.from_words(ctx, a, sc), fh.SlotVector.from_words(ctx, b, sc)
    assert np.array_equal(fh.rotate(x, 3).words(), orc.rotate(a, 3, orc.rotation_key(3)))
    if limbs > 1:
        assert np.array_equal(fh.mult_cipher(x, y).words(), orc.mult_cipher(a, b, orc.relin_key()))
        want = orc.rotate_sum([a, b], [3, -9], [orc.rotation_key(3), orc.rotation_key(-9)])
        assert np.array_equal(fh.rotate_sum([x, y], [3, -9]).words(), want)


def test_secure_sse_keys_bit_exact(secure):
    ctx, orc, _ = secure
    assert np.array_equal(ctx.download_key(2), orc.keygen(2))
    assert np.array_equal(ctx.download_key(4), orc.keygen(4))


def test_secure_bootstrap_precision(secure):
    """Full-slot bootstrapping through the sparse-secret encapsulation at the
    headline chain: lands on the depth budget within 1e-4."""
    ctx, _, _ = secure
    v = np.random.default_rng(31).uniform(-1, 1, ctx.slots())
    x = fh.level_down(fh.SlotVector.encode(ctx, v), 1)
    y = fh.bootstrap(x)
    assert y.level() == ctx.depth_budget() == 12
    assert np.abs(y.slots() - v).max() < 1e-4
