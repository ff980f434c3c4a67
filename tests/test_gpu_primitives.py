"""GPU parity: every RNS-CKKS primitive of the sm_100a engine is bit-exact
against the CPU oracle (oracle/ckks_oracle.c) on identical inputs and keys.

Mirrors the reference's backend tests (proj/tests/test_backend.cpp:80-220:
rotation direction/range, level rules, depth exhaustion) at the RNS level.
"""
import numpy as np
import pytest

import paper_2510_03996_b200 as fh
from oracle.ckks_oracle import Oracle

pytestmark = pytest.mark.gpu

SMALL = dict(logN=12, L=6, K=2, dnum=3, first=50, scale=40, special=60, seed=11)


def make_pair(logN, L, K, dnum, first, scale, special, seed, depth=None, digit_split=0):
    cfg = fh.ContextConfig(1 << logN, 1 << (logN - 1), depth if depth is not None else L - 1,
                           fh.CryptoMetadata(first, scale, dnum), limbs=L, special_limbs=K, special_bits=special,
                           seed=seed, digit_split=digit_split, allow_insecure=True)
    ctx = fh.SlotContext(cfg)
    orc = Oracle(logN, L, K, dnum, first, scale, special, seed, digit_split=digit_split)
    return ctx, orc


@pytest.fixture(scope="module")
def small():
    return make_pair(**SMALL)


def rand_limbs(orc, nlimbs, rng, primes_idx=None):
    idx = primes_idx if primes_idx is not None else range(nlimbs)
    return np.stack([rng.integers(0, int(orc.primes[i]), orc.N, dtype=np.uint64) for i in idx])


def test_params_match_oracle(small):
    ctx, orc = small
    assert (ctx.primes == orc.primes).all()
    assert np.array_equal(ctx.scales, orc.T)


@pytest.mark.parametrize("logN", [10, 11, 12, 13, 14, 15, 16])
def test_ntt_bit_exact_all_sizes(logN):
    ctx, orc = make_pair(logN, 3, 2, 3, 50, 40, 60, 5)
    rng = np.random.default_rng(logN)
    a = rand_limbs(orc, 5, rng)  # q0..q2, p0, p1 as one 5-limb poly (limb i uses prime i)
    fwd = ctx.ntt(a)
    want = orc.ntt_limbs(a)
    assert np.array_equal(fwd, want)
    back = ctx.ntt(fwd, inverse=True)
    assert np.array_equal(back, a)
    assert np.array_equal(back, orc.ntt_limbs(want, inverse=True))


def test_ntt_batched_polys(small):
    ctx, orc = small
    rng = np.random.default_rng(1)
    a = np.stack([rand_limbs(orc, 4, rng) for _ in range(3)])
    got = ctx.ntt(a)
    for p in range(3):
        assert np.array_equal(got[p], orc.ntt_limbs(a[p]))


@pytest.mark.parametrize("t", [1, 2, 5, -1, -7, 1000, 2047])
def test_automorphism_bit_exact(small, t):
    ctx, orc = small
    rng = np.random.default_rng(t % 97)
    a = rand_limbs(orc, 4, rng)
    g = orc.galois(t)
    assert ctx.galois_element(t) == g
    assert np.array_equal(ctx.automorph(a, g), orc.automorph_ntt(a, g))


def test_keygen_bit_exact(small):
    ctx, orc = small
    g = orc.galois(3)
    assert np.array_equal(ctx.download_key(g), orc.keygen(g))
    assert np.array_equal(ctx.download_key(0), orc.keygen(0))


def test_encrypt_bit_exact_and_decrypt(small):
    ctx, orc = small
    rng = np.random.default_rng(2)
    vals = rng.uniform(-1, 1, orc.S)
    ct = fh.SlotVector.encode_top(ctx, vals)
    # the engine's encryption counter starts at 0 and increments per encryption
    want = None
    for counter in range(0, 64):
        cand = orc.encrypt(vals, counter)
        if np.array_equal(cand[1], ct.words()[1]):
            want = cand
            break
    assert want is not None, "no matching encryption counter"
    assert np.array_equal(ct.words(), want)
    assert np.abs(ct.slots() - vals).max() < 1e-6
    assert np.abs(orc.decrypt(want, orc.T[-1]) - vals).max() < 1e-6


def _oracle_ct(orc, rng, counter=5):
    vals = rng.uniform(-1, 1, orc.S)
    return vals, orc.encrypt(vals, counter)


@pytest.mark.parametrize("t", [1, -1, 3, 64, -1000, 2047])
def test_rotation_bit_exact(small, t):
    ctx, orc = small
    rng = np.random.default_rng(100 + abs(t))
    vals, ct = _oracle_ct(orc, rng)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.rotate(x, t)
    want = orc.rotate(ct, t, orc.rotation_key(t))
    assert np.array_equal(got.words(), want)
    assert np.abs(got.slots() - np.roll(vals, -t)).max() < 1e-6
    assert got.level() == x.level()


@pytest.mark.parametrize("limbs", [6, 4, 3, 1])
def test_rotation_lower_levels(small, limbs):
    ctx, orc = small
    rng = np.random.default_rng(limbs)
    vals, ct = _oracle_ct(orc, rng)
    ct = np.ascontiguousarray(ct[:, :limbs])
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.rotate(x, 7)
    want = orc.rotate(ct, 7, orc.rotation_key(7))
    assert np.array_equal(got.words(), want)


def test_hoisted_equals_single(small):
    ctx, orc = small
    rng = np.random.default_rng(9)
    vals, ct = _oracle_ct(orc, rng)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    ts = [1, 2, 3, 28, 29, -5]
    hs = fh.rotate_hoisted(x, ts)
    for t, h in zip(ts, hs):
        assert np.array_equal(h.words(), fh.rotate(x, t).words())
        assert np.array_equal(h.words(), orc.rotate(ct, t, orc.rotation_key(t)))


@pytest.mark.parametrize("ts", [[1, -1], [3, 64, -1000, 2047, 5], [0, 7, 7]])
def test_rotate_sum_bit_exact(small, ts):
    """rotate-and-sum (one ModDown per output, c0 folded in as P * c0) is
    bit-exact against the oracle's restatement ock_rotate_sum; identity terms
    are added directly."""
    ctx, orc = small
    rng = np.random.default_rng(300 + len(ts))
    cts = [_oracle_ct(orc, rng, counter=20 + i)[1] for i in range(len(ts))]
    if len(ts) == 3:
        cts[2] = cts[1]  # repeated input: shared ModUp
    xs = [fh.SlotVector.from_words(ctx, c, orc.T[-1]) for c in cts]
    got = fh.rotate_sum(xs, ts).words()
    ks = [(c, t) for c, t in zip(cts, ts) if orc.galois(t) != 1]
    want = orc.rotate_sum([c for c, _ in ks], [t for _, t in ks], [orc.rotation_key(t) for _, t in ks])
    for c, t in zip(cts, ts):
        if orc.galois(t) == 1:
            want = orc.add(want, c)
    assert np.array_equal(got, want)


def test_keyswitch_modup_moddown(small):
    ctx, orc = small
    rng = np.random.default_rng(4)
    _, ct = _oracle_ct(orc, rng)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    g = orc.galois(5)
    got = fh.keyswitch_raw(x, g, g).words()
    ks0, ks1 = orc.keyswitch(ct[1], orc.keygen(g), g)
    assert np.array_equal(got[0], ks0)
    assert np.array_equal(got[1], ks1)


def test_rescale_bit_exact(small):
    ctx, orc = small
    rng = np.random.default_rng(5)
    a = np.stack([rand_limbs(orc, 6, rng), rand_limbs(orc, 6, rng)])
    x = fh.SlotVector.from_words(ctx, a, 1.0)
    assert np.array_equal(fh.rescale(x).words(), orc.rescale(a))


def test_mult_plain_bit_exact(small):
    ctx, orc = small
    rng = np.random.default_rng(6)
    vals, ct = _oracle_ct(orc, rng)
    pv = rng.uniform(-1, 1, orc.S)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.mult_plain(x, pv)
    want, s = orc.mult_plain(ct, orc.T[-1], pv)
    assert np.array_equal(got.words(), want)
    assert got.scale() == s
    assert got.level() == x.level() - 1
    assert np.abs(got.slots() - vals * pv).max() < 1e-6


def test_mult_const_bit_exact(small):
    ctx, orc = small
    rng = np.random.default_rng(7)
    vals, ct = _oracle_ct(orc, rng)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.mult_plain(x, np.full(orc.S, -0.3125))
    want, _ = orc.mult_plain(ct, orc.T[-1], np.full(orc.S, -0.3125))
    assert np.array_equal(got.words(), want)


def test_mult_cipher_bit_exact(small):
    ctx, orc = small
    rng = np.random.default_rng(8)
    va, ca = _oracle_ct(orc, rng, 1)
    vb, cb = _oracle_ct(orc, rng, 2)
    a = fh.SlotVector.from_words(ctx, ca, orc.T[-1])
    b = fh.SlotVector.from_words(ctx, cb, orc.T[-1])
    got = fh.mult_cipher(a, b)
    want = orc.mult_cipher(ca, cb, orc.relin_key())
    assert np.array_equal(got.words(), want)
    assert got.level() == a.level() - 1
    assert np.abs(got.slots() - va * vb).max() < 1e-6


def test_level_down_bit_exact(small):
    ctx, orc = small
    rng = np.random.default_rng(10)
    vals, ct = _oracle_ct(orc, rng)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.level_down(x, 3)
    want, s = orc.level_down(ct, orc.T[-1], 3)
    assert np.array_equal(got.words(), want)
    assert got.scale() == s
    assert np.abs(got.slots() - vals).max() < 1e-6


def test_add_sub_levels_and_values(small):
    ctx, _ = small
    rng = np.random.default_rng(11)
    va, vb = rng.uniform(-1, 1, ctx.slots()), rng.uniform(-1, 1, ctx.slots())
    a = fh.SlotVector.encode(ctx, va)
    b = fh.mult_plain(fh.SlotVector.encode(ctx, vb), np.full(ctx.slots(), 1.0))
    s = fh.add(a, b)
    d = fh.sub(a, b)
    assert s.level() == min(a.level(), b.level())
    assert np.abs(s.slots() - (va + vb)).max() < 1e-6
    assert np.abs(d.slots() - (va - vb)).max() < 1e-6


def test_rotation_range_errors(small):
    ctx, _ = small
    x = fh.SlotVector.encode(ctx, [1.0, 2.0])
    S = ctx.slots()
    with pytest.raises(fh.InvalidRotationError):
        fh.rotate(x, S)
    with pytest.raises(fh.InvalidRotationError):
        fh.rotate(x, -S)
    fh.rotate(x, S - 1)
    fh.rotate(x, -(S - 1))


def test_depth_exhaustion(small):
    ctx, _ = small
    x = fh.SlotVector.encode(ctx, [0.5])
    ones = np.ones(ctx.slots())
    while x.level() > 0:
        x = fh.mult_plain(x, ones)
    with pytest.raises(fh.DepthExhaustedError):
        fh.mult_plain(x, ones)
    with pytest.raises(fh.DepthExhaustedError):
        fh.mult_cipher(x, x)


def test_trace_events(small):
    ctx, _ = small
    rec = ctx.attach_recorder()
    x = fh.SlotVector.encode(ctx, [1.0, 2.0, 3.0])
    y = fh.rotate(x, 2)
    z = fh.mult_plain(y, np.ones(ctx.slots()) * 2)
    fh.mult_cipher(z, z)
    ev = rec.snapshot()
    assert [(e.kind, e.value) for e in ev] == [("rotation", 2), ("mult_plain", x.level() - 1),
                                               ("mult_cipher", x.level() - 2)]
    ctx.detach_recorder()


@pytest.mark.slow
def test_config2_rotation_bit_exact():
    """BASELINE configs[1] parameters: N=2^16, L=24, K=8, dnum=3."""
    ctx, orc = make_pair(16, 24, 8, 3, 60, 50, 60, 2001)
    rng = np.random.default_rng(2001)
    vals, ct = _oracle_ct(orc, rng)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.rotate(x, 1)
    assert np.array_equal(got.words(), orc.rotate(ct, 1, orc.rotation_key(1)))
    got = fh.rescale(x)
    assert np.array_equal(got.words(), orc.rescale(ct))


def test_config1_rotation_bit_exact():
    """BASELINE configs[0] parameters: N=2^14, 50-bit q0, 40-bit scaling, L=11, dnum=3."""
    ctx, orc = make_pair(14, 11, 4, 3, 50, 40, 60, 1001)
    rng = np.random.default_rng(1001)
    vals, ct = _oracle_ct(orc, rng)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    got = fh.rotate(x, 28)
    assert np.array_equal(got.words(), orc.rotate(ct, 28, orc.rotation_key(28)))
    assert np.abs(got.slots() - np.roll(vals, -28)).max() < 1e-6


@pytest.mark.parametrize("L,t", [(7, 3), (9, -17), (13, 100)])
def test_balanced_digits_keyswitch_bit_exact(L, t):
    """Key-switching digits balanced by prime bit size (60-bit q0, 40-bit rest:
    unequal limb counts per digit): keys, rotation and rotate-and-sum stay
    bit-exact against the oracle's restatement (ock_set_digit_split)."""
    ctx, orc = make_pair(12, L, 4, 3, 60, 40, 60, 23, digit_split=1)
    rng = np.random.default_rng(L)
    vals, ct = _oracle_ct(orc, rng, counter=40)
    x = fh.SlotVector.from_words(ctx, ct, orc.T[-1])
    g = orc.galois(t)
    assert np.array_equal(ctx.download_key(g), orc.keygen(g))
    assert np.array_equal(fh.rotate(x, t).words(), orc.rotate(ct, t, orc.rotation_key(t)))
    for limbs in (L - 2, 3):  # lower levels: fewer active digits
        xs = fh.level_down(x, limbs)
        c2 = xs.words()
        assert np.array_equal(fh.rotate(xs, t).words(), orc.rotate(c2, t, orc.rotation_key(t)))
    y = fh.rotate_sum([x, x], [t, 1])
    want = orc.rotate_sum([ct, ct], [t, 1], [orc.rotation_key(t), orc.rotation_key(1)])
    assert np.array_equal(y.words(), want)



def test_async_transfers_bit_exact(small):
    """Asynchronous copy streams: uploads / downloads of several ciphertexts
    overlapping compute give the same words as the blocking path."""
    ctx, orc = small
    rng = np.random.default_rng(77)
    cts = [_oracle_ct(orc, rng, counter=60 + i)[1] for i in range(4)]
    outs = [np.zeros_like(c) for c in cts]
    for rep in range(2):
        xs = [fh.SlotVector.from_words(ctx, c, orc.T[-1], async_copy=True) for c in cts]
        ys = fh.rotate_many(xs, [1, 3, -2, 5])
        for y, o in zip(ys, outs):
            y.words(out=o, async_copy=True)
        ctx.wait_transfers()
        for c, t, o in zip(cts, [1, 3, -2, 5], outs):
            assert np.array_equal(o, orc.rotate(c, t, orc.rotation_key(t)))


@pytest.mark.parametrize("limbs", [1, 4, 6])
def test_packed_transfers_bit_exact(small, limbs):
    """Packed wire format (fheon_ct_*_packed): the device packs to exactly the
    oracle's bitstream and unpacks it back to the same words (sync and async)."""
    ctx, orc = small
    rng = np.random.default_rng(90 + limbs)
    ct = _oracle_ct(orc, rng, counter=70)[1][:, :limbs].copy()
    packed = orc.pack(ct)
    assert ctx.packed_words(limbs) == packed.size
    x = fh.SlotVector.from_packed(ctx, packed, limbs, orc.T[limbs - 1])
    assert np.array_equal(x.words(), ct)
    assert np.array_equal(fh.SlotVector.from_words(ctx, ct, orc.T[limbs - 1]).packed(), packed)
    out = np.zeros(packed.size, np.uint64)
    y = fh.SlotVector.from_packed(ctx, packed, limbs, orc.T[limbs - 1], async_copy=True)
    y.packed(out=out, async_copy=True)
    ctx.wait_transfers()
    assert np.array_equal(out, packed)


def test_packed_transfers_config2_roundtrip():
    """BASELINE configs[1] size (N=2^16, 60 + 23 x 50-bit limbs): packed size
    0.79 of the raw words, device pack/unpack round trip bit-exact on a rotated
    ciphertext (size-independent property: unpack(pack(x)) == x)."""
    cfg = fh.ContextConfig(1 << 16, 1 << 15, 23, fh.CryptoMetadata(60, 50, 3), limbs=24, special_limbs=8,
                           special_bits=60, seed=2001)
    ctx = fh.SlotContext(cfg)
    x = fh.rotate(fh.SlotVector.encode_top(ctx, np.random.default_rng(3).uniform(-1, 1, 1 << 15)), 5)
    w = x.words()
    p = x.packed()
    bits = sum(int(q).bit_length() for q in ctx.primes[:24])
    assert bits <= 60 + 23 * 51 and p.size == 2 * (1 << 16) * bits // 64
    assert np.array_equal(fh.SlotVector.from_packed(ctx, p, 24, x.scale()).words(), w)


@pytest.mark.parametrize("shared", [True, False])
def test_rotate_sum_many_groups_bit_exact(small, shared):
    """Several rotate-and-sum groups in one pipeline.  shared=True: every group
    rotates ONE input under the same key list -- the hoisted-stage kernel
    (k_ks_inner_shared, every key slice read once per launch); False: distinct
    key lists per group (k_ks_inner_sum).  Each output bit-exact against the
    oracle's ock_rotate_sum."""
    ctx, orc = small
    rng = np.random.default_rng(410 + shared)
    cts = [_oracle_ct(orc, rng, counter=80 + i)[1] for i in range(3)]
    xs = [fh.SlotVector.from_words(ctx, c, orc.T[-1]) for c in cts]
    lists = [[1, 3, -2]] * 3 if shared else [[1, 3, -2], [5, -1], [2, 7, 11, -9]]
    outs = fh.rotate_sum_many([[(x, t) for t in ts] for x, ts in zip(xs, lists)])
    for c, ts, o in zip(cts, lists, outs):
        want = orc.rotate_sum([c] * len(ts), ts, [orc.rotation_key(t) for t in ts])
        assert np.array_equal(o.words(), want)
