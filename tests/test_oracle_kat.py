"""CPU: pins the RNS-CKKS oracle (oracle/ckks_oracle.c) with known-answer
tests against definitions: the reference has no RNS
arithmetic, so each primitive is checked against its mathematical definition
with independent Python big-integer code.
"""
import numpy as np
import pytest

from oracle.ckks_oracle import Oracle


@pytest.fixture(scope="module")
def tiny():
    return Oracle(5, 4, 2, 2, 50, 40, 55, seed=7)  # N = 32: O(N^2) checks are cheap


@pytest.fixture(scope="module")
def small():
    return Oracle(10, 6, 2, 3, 50, 40, 60, seed=11)


def _bits(q):
    return int(q).bit_length()


def test_prime_chain_properties(small):
    o = small
    M = 2 * o.N
    ps = [int(p) for p in o.primes]
    assert len(set(ps)) == len(ps)
    for p in ps:
        assert p % M == 1
        assert all(pow(b, p - 1, p) == 1 for b in (2, 3, 5, 7))
    assert _bits(ps[0]) == 50
    assert all(_bits(p) in (40, 41) for p in ps[1:o.L])
    assert all(_bits(p) == 60 for p in ps[o.L:])
    # FLEXIBLEAUTO targets: T_{l-1} = T_l^2 / q_l, all within 2^-12 of 2^40
    T = o.T
    for lv in range(o.L - 1, 0, -1):
        assert T[lv - 1] == (T[lv] * T[lv]) / float(ps[lv])
    assert np.all(np.abs(T / 2.0 ** 40 - 1) < 2 ** -12)


def test_psi_is_primitive_2n_root(small):
    o = small
    for q, psi in zip(o.primes, o.psi):
        q, psi = int(q), int(psi)
        assert pow(psi, o.N, q) == q - 1
        assert pow(psi, 2 * o.N, q) == 1


def test_ntt_matches_naive_evaluation(tiny):
    o = tiny
    rng = np.random.default_rng(0)
    for pi in range(o.L + o.K):
        a = rng.integers(0, int(o.primes[pi]), o.N, dtype=np.uint64)
        assert np.array_equal(o.ntt(a, pi), o.ntt_naive(a, pi))
        # independent big-int definition: out[i] = a(psi^(2 brv(i) + 1))
        q, psi = int(o.primes[pi]), int(o.psi[pi])
        lg = o.logN
        i = 5
        e = 2 * int(format(i, f"0{lg}b")[::-1], 2) + 1
        x = pow(psi, e, q)
        want = sum(int(c) * pow(x, k, q) for k, c in enumerate(a)) % q
        assert int(o.ntt(a, pi)[i]) == want


def test_ntt_roundtrip_and_convolution(small):
    o = small
    rng = np.random.default_rng(1)
    for pi in (0, 3, o.L):
        q = int(o.primes[pi])
        a = rng.integers(0, q, o.N, dtype=np.uint64)
        b = rng.integers(0, q, o.N, dtype=np.uint64)
        assert np.array_equal(o.intt(o.ntt(a, pi), pi), a)
        pa, pb = o.ntt(a, pi).astype(object), o.ntt(b, pi).astype(object)
        prod = np.array([(x * y) % q for x, y in zip(pa, pb)], dtype=np.uint64)
        assert np.array_equal(o.intt(prod, pi), o.negacyclic_mul_naive(a, b, pi))


def test_automorphism_definition(small):
    o = small
    rng = np.random.default_rng(2)
    a = np.stack([rng.integers(0, int(o.primes[i]), o.N, dtype=np.uint64) for i in range(3)])
    for t in (1, 2, 7, -1, -5):
        g = o.galois(t)
        assert g == pow(5, t % o.S, 2 * o.N)
        coeff = o.automorph_coeff(a, g)
        # X^k -> (-1)^{floor(kg/N)} X^{kg mod N}
        for k in (0, 1, 17, o.N - 1):
            kg = k * g % (2 * o.N)
            dst, neg = kg % o.N, kg >= o.N
            for l in range(3):
                q = int(o.primes[l])
                v = int(a[l][k])
                assert int(coeff[l][dst]) == ((q - v) % q if neg else v)
        assert np.array_equal(o.automorph_ntt(o.ntt_limbs(a), g), o.ntt_limbs(coeff))


def test_encoder_canonical_embedding(tiny):
    o = tiny
    rng = np.random.default_rng(3)
    vals = rng.uniform(-1, 1, o.S)
    scale = 2.0 ** 30
    m = o.encode_coeffs(vals, scale)
    zeta = np.exp(2j * np.pi / (2 * o.N))
    for j in range(o.S):
        e = pow(5, j, 2 * o.N)
        v = sum(int(m[k]) * zeta ** (e * k) for k in range(o.N)) / scale
        assert abs(v - vals[j]) < 1e-7
    assert np.abs(o.decode_coeffs(m.astype(np.float64), scale) - vals).max() < 2 ** -25


def test_encoder_roundtrip_2e30(small):
    o = small
    rng = np.random.default_rng(4)
    vals = rng.uniform(-1, 1, o.S)
    m = o.encode_coeffs(vals, 2.0 ** 40)
    assert np.abs(o.decode_coeffs(m.astype(np.float64), 2.0 ** 40) - vals).max() < 2 ** -30


def test_encrypt_decrypt(small):
    o = small
    rng = np.random.default_rng(5)
    vals = rng.uniform(-1, 1, o.S)
    ct = o.encrypt(vals, 3)
    assert np.abs(o.decrypt(ct, o.T[-1]) - vals).max() < 1e-7
    # encryption is deterministic in (seed, counter) and differs across counters
    assert np.array_equal(ct, o.encrypt(vals, 3))
    assert not np.array_equal(ct[1], o.encrypt(vals, 4)[1])


def test_rescale_is_rounded_division_crt(small):
    """rescale == round(x / q_l) per coefficient, verified by exact CRT."""
    o = small
    rng = np.random.default_rng(6)
    limbs = 4
    qs = [int(q) for q in o.primes[:limbs]]
    Q = int(np.prod(np.array(qs, dtype=object)))
    X = [int(x) for x in rng.integers(0, 2 ** 62, o.N)]
    X = [(x * 12345678901 + 987654321) % Q for x in X]
    coeff = np.array([[x % q for x in X] for q in qs], dtype=np.uint64)
    ntt = o.ntt_limbs(coeff)
    ct = np.stack([ntt, ntt])
    out = o.rescale(ct)
    back = o.ntt_limbs(out[0], inverse=True)
    ql = qs[-1]
    for k in range(0, o.N, 37):
        x = X[k]
        xc = x if x <= Q // 2 else x - Q  # centred representative
        want = (xc - (((xc % ql) + ql // 2) % ql - ql // 2)) // ql  # = round(xc / ql)
        for i in range(limbs - 1):
            assert int(back[i][k]) == want % qs[i]


def test_rotation_decrypts_to_left_shift(small):
    """rotation direction of the reference: out[j] = in[(j + t) mod S] (kernels.hpp:26)."""
    o = small
    rng = np.random.default_rng(7)
    vals = rng.uniform(-1, 1, o.S)
    ct = o.encrypt(vals, 1)
    for t in (1, 3, -2, o.S - 1):
        r = o.rotate(ct, t, o.rotation_key(t))
        assert np.abs(o.decrypt(r, o.T[-1]) - np.roll(vals, -t)).max() < 1e-6


def test_rotate_sum_decrypts_to_sum_of_shifts(small):
    """rotate-and-sum with one ModDown (ock_rotate_sum) = sum of left shifts, with
    no more noise than separate rotations followed by additions."""
    o = small
    rng = np.random.default_rng(17)
    v1, v2 = rng.uniform(-1, 1, o.S), rng.uniform(-1, 1, o.S)
    c1, c2 = o.encrypt(v1, 3), o.encrypt(v2, 4)
    ts = [3, -7, 5, 0]
    cts = [c1, c2, c1, c2]
    out = o.rotate_sum(cts[:3], ts[:3], [o.rotation_key(t) for t in ts[:3]])
    want = np.roll(v1, -3) + np.roll(v2, 7) + np.roll(v1, -5)
    err = np.abs(o.decrypt(out, o.T[-1]) - want).max()
    sep = o.add(o.add(o.rotate(c1, 3, o.rotation_key(3)), o.rotate(c2, -7, o.rotation_key(-7))),
                o.rotate(c1, 5, o.rotation_key(5)))
    err_sep = np.abs(o.decrypt(sep, o.T[-1]) - want).max()
    assert err < 1e-6 and err <= 2 * err_sep


def test_keyswitch_noise_bound(small):
    o = small
    rng = np.random.default_rng(8)
    ct = o.encrypt(rng.uniform(-1, 1, o.S), 2)
    s = o.secret().astype(np.int64)
    g = o.galois(5)
    ks0, ks1 = o.keyswitch(ct[1], o.keygen(g), g)
    q = int(o.primes[0])
    s_ntt = o.ntt(np.array([x % q for x in s], dtype=np.uint64), 0).astype(object)
    sp = o.automorph_ntt(s_ntt.astype(np.uint64)[None, :], g)[0].astype(object)
    d = o.automorph_ntt(ct[1][:1], g)[0].astype(object)
    err = (ks0[0].astype(object) + ks1[0].astype(object) * s_ntt - d * sp) % q
    e = o.intt(np.array(err, dtype=np.uint64), 0).astype(object)
    e = np.array([x - q if x > q // 2 else x for x in e], dtype=np.float64)
    # ModDown rounding (|u| <= 1/2 each) times ||s||_1 plus key noise / P: tiny
    assert np.abs(e).max() < 200
    assert abs(e.mean()) < 5


def test_mult_plain_cipher_and_level_down(small):
    o = small
    rng = np.random.default_rng(9)
    a, b = rng.uniform(-1, 1, o.S), rng.uniform(-1, 1, o.S)
    ca, cb = o.encrypt(a, 10), o.encrypt(b, 11)
    mp, s = o.mult_plain(ca, o.T[-1], b)
    assert s == o.T[-2]
    assert np.abs(o.decrypt(mp, s) - a * b).max() < 1e-6
    mc = o.mult_cipher(ca, cb, o.relin_key())
    assert np.abs(o.decrypt(mc, o.T[-1] ** 2 / float(o.primes[o.L - 1])) - a * b).max() < 1e-6
    ld, s2 = o.level_down(ca, o.T[-1], 2)
    assert ld.shape[1] == 2
    assert np.abs(o.decrypt(ld, s2) - a).max() < 1e-6


def test_constant_plaintext_is_degree_zero(small):
    o = small
    m = o.encode_coeffs(np.full(o.S, 0.375), 2.0 ** 40)
    assert m[0] == round(0.375 * 2 ** 40) and not m[1:].any()


def test_packed_wire_format_definition(small):
    """oracle pack == the definition with Python big integers: limb streams of
    bit_length(q_i) bits per canonical word, concatenated little-endian
    (N >= 1024, as the engine requires, so every limb stream is whole words)."""
    o = small
    rng = np.random.default_rng(5)
    limbs = 3
    ct = np.stack([np.stack([rng.integers(0, int(o.primes[i]), o.N, dtype=np.uint64) for i in range(limbs)])
                   for _ in range(2)])
    big, pos = 0, 0
    for p in range(2):
        for i in range(limbs):
            b = _bits(o.primes[i])
            for v in ct[p, i]:
                big |= int(v) << pos
                pos += b
    words = o.pack(ct)
    assert words.size * 64 == pos and pos == 2 * o.N * sum(_bits(o.primes[i]) for i in range(limbs))
    assert [int(w) for w in words] == [(big >> (64 * k)) & ((1 << 64) - 1) for k in range(words.size)]
    assert np.array_equal(o.unpack(words, limbs), ct)


def test_packed_wire_format_extremes(small):
    """all-zero and all-(q_i - 1) words survive the round trip (no bit bleeds
    into the neighbouring coefficient)."""
    o = small
    for limbs in (1, 6):
        top = np.stack([np.stack([np.full(o.N, int(o.primes[i]) - 1, np.uint64) for i in range(limbs)])
                        for _ in range(2)])
        for ct in (np.zeros_like(top), top):
            assert np.array_equal(o.unpack(o.pack(ct), limbs), ct)
