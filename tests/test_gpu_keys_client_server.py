"""Evaluation-key serialization and a secret-free SERVER context (SURVEY 8(b)
"keygen / key upload", 8(f) item 4; PAPER.md:541-566 serialized keys): the
client generates keys and ciphertexts, ships them in the packed wire format;
the server (ContextConfig.no_secret -- it never holds the secret) uploads the
keys and computes; the client decrypts.  The server's results are bit-exact
with the same ops run on the client."""
import dataclasses

import numpy as np
import pytest

import paper_2510_03996_b200 as fh

pytestmark = pytest.mark.gpu

N, S = 1 << 12, 1 << 11


def _cfg(**kw):
    base = fh.ContextConfig(N, S, 6, fh.CryptoMetadata(55, 40, 3), limbs=7, special_limbs=3, special_bits=60,
                            seed=41, allow_insecure=True)
    return dataclasses.replace(base, **kw)


def test_key_packed_roundtrip_and_server_compute():
    client = fh.SlotContext(_cfg())
    server = fh.SlotContext(_cfg(no_secret=True))
    assert (client.primes == server.primes).all()
    rng = np.random.default_rng(5)
    a, b = rng.uniform(-1, 1, S), rng.uniform(-1, 1, S)
    xa, xb = fh.SlotVector.encode(client, a), fh.SlotVector.encode(client, b)
    ts = [1, -7, 100]
    client.keygen_rotations(ts)
    client.keygen_relin()
    ids = [client.galois_element(t) for t in ts] + [0]
    pw = client.key_packed_words()
    L, K, dnum = 7, 3, 3
    bits = sum(int(q).bit_length() for q in client.primes[:L + K])
    assert pw == dnum * 2 * N * bits // 64  # 2 dnum polys of L+K limbs at b_i bits each
    for i in ids:
        server.key_upload(i, client.key_download_packed(i))
        assert np.array_equal(server.download_key(i), client.download_key(i))  # bit-exact key transfer
    assert server.key_uploads()["uploads"] == len(ids)
    sa = fh.SlotVector.from_packed(server, xa.packed(), xa.limbs(), xa.scale())
    sb = fh.SlotVector.from_packed(server, xb.packed(), xb.limbs(), xb.scale())
    ys = fh.rotate_many([sa, sa, sb], ts)
    z = fh.mult_cipher(fh.add(ys[0], ys[2]), sb)
    want = fh.mult_cipher(fh.add(fh.rotate(xa, 1), fh.rotate(xb, 100)), xb)
    assert np.array_equal(z.words(), want.words())  # server == client, bit for bit
    back = fh.SlotVector.from_packed(client, z.packed(), z.limbs(), z.scale())
    assert np.abs(back.slots() - (np.roll(a, -1) + np.roll(b, -100)) * b).max() < 1e-4
    with pytest.raises(fh.Error, match="no secret"):
        fh.SlotVector.encode(server, a)
    with pytest.raises(fh.Error, match="no secret"):
        sa.slots()
    with pytest.raises(fh.Error, match="not resident"):
        fh.rotate(sa, 3)  # a key the client never sent


def test_server_bootstraps_with_uploaded_keys():
    """Bootstrapping on a server context: the client uploads exactly the ids the
    server lists (relinearisation, conjugation, CtS / StC rotations, the
    sparse-secret encapsulation keys) asynchronously on the upload stream."""
    cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=24, special_limbs=8, special_bits=60,
                           seed=43, bootstrap=True, boot_scale_bits=55, allow_insecure=True)
    client = fh.SlotContext(cfg)
    server = fh.SlotContext(dataclasses.replace(cfg, no_secret=True))
    need = server.required_key_ids()
    assert 0 in need and 2 in need and 4 in need and len(need) > 10
    assert sorted(need) == sorted(client.required_key_ids())
    import torch
    host = {}
    for i in need:
        buf = torch.empty(client.key_packed_words(), dtype=torch.uint64, pin_memory=True).numpy()
        host[i] = client.key_download_packed(i, out=buf)
    for i in need:
        server.key_upload(i, host[i], async_copy=True)
    server.wait_transfers()
    v = np.random.default_rng(9).uniform(-1, 1, S)
    x = fh.level_down(fh.SlotVector.encode(client, v), 1)
    sx = fh.SlotVector.from_packed(server, x.packed(), x.limbs(), x.scale())
    sy = fh.bootstrap(sx)
    y = fh.SlotVector.from_packed(client, sy.packed(), sy.limbs(), sy.scale())
    assert y.level() == client.depth_budget()
    assert np.abs(y.slots() - v).max() < 1e-4
    assert np.array_equal(sy.words(), fh.bootstrap(fh.SlotVector.from_words(client, x.words(), x.scale())).words())


def test_key_sharing_clone_runs_concurrently_bit_exact():
    """SlotContext.clone: a second context over the same keys (no new key memory),
    own stream; two host threads drive both at once and each result is bit-exact
    with the same ops on the parent alone."""
    import threading
    cfg = fh.ContextConfig(N, S, -1, fh.CryptoMetadata(55, 40, 3), limbs=24, special_limbs=8, special_bits=60,
                           seed=47, bootstrap=True, boot_scale_bits=55, allow_insecure=True)
    parent = fh.SlotContext(cfg)
    parent.keygen_rotations([1, 5])
    kb = parent.key_bytes()
    twin = parent.clone()
    assert twin.key_bytes() == kb and twin.key_count() == parent.key_count()
    v = np.random.default_rng(3).uniform(-1, 1, S)
    x = fh.level_down(fh.SlotVector.encode(parent, v), 1)
    words, scale = x.words(), x.scale()

    def pipeline(ctx):
        y = fh.SlotVector.from_words(ctx, words, scale)
        y = fh.bootstrap(y)
        return fh.mult_cipher(fh.rotate(y, 1), fh.rotate(y, 5)).words()

    want = pipeline(parent)
    got = {}
    th = [threading.Thread(target=lambda c, k: got.__setitem__(k, pipeline(c)), args=(c, k))
          for k, c in (("a", parent), ("b", twin))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert np.array_equal(got["a"], want) and np.array_equal(got["b"], want)
    assert twin.key_bytes() == kb  # nothing was generated on the clone
