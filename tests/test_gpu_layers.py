"""GPU parity of the layer API against the reference's own layer algorithms.

The checker is the UNMODIFIED reference slotcnn core (oracle/_ref, built from
/root/reference/proj): the same inputs are run through its cleartext slot
simulator and through the encrypted B200 engine; the decrypted slots must
agree within max-abs 1e-3 (the north-star tolerance), the output level must
be identical and the trace (rotation indices, mult level_after, in order)
must be identical.  Case generation follows acceptance criterion 1
(proj/tests/acceptance.cpp:226-426): W in {4,6,8}, C,F in 1..4, random
kernel/stride/padding, both striding flavours, degrees {7,27,59}.
"""
import numpy as np
import pytest

import paper_2510_03996_b200 as fh
from oracle import ref as sref

pytestmark = pytest.mark.gpu

TOL = 1e-3
LOGN, DEPTH = 12, 13


@pytest.fixture(scope="module", params=["reference", "fast"])
def env(request):
    """Both rotation schedules: "reference" must replay the reference's trace
    multiset exactly; "fast" (the default) must give the same slots and levels."""
    cfg = fh.ContextConfig(1 << LOGN, 1 << (LOGN - 1), DEPTH, fh.CryptoMetadata(52, 40, 3), limbs=DEPTH + 1,
                           special_limbs=4, special_bits=60, seed=9001, schedule=request.param,
                           allow_insecure=True)
    ctx = fh.SlotContext(cfg)
    return ctx, sref.Ref(1 << LOGN, 1 << (LOGN - 1), DEPTH)


def run_both(ctx, fn_gpu, fn_ref, x):
    rec = ctx.attach_recorder()
    xs = fh.SlotVector.encode(ctx, np.asarray(x).reshape(-1))
    out = fn_gpu(xs)
    ev = [(e.kind, e.value) for e in rec.snapshot()]
    ctx.detach_recorder()
    r = fn_ref(np.asarray(x).reshape(-1))
    return out, ev, r


def check(out_ct, ev, r, tag, schedule="reference"):
    got = out_ct.slots()
    err = np.abs(got - r.slots).max()
    assert err < TOL, f"{tag}: max abs error {err}"
    assert out_ct.level() == r.level, f"{tag}: level {out_ct.level()} vs reference {r.level}"
    if schedule == "reference":
        # identical event multiset (rotation indices with counts, mult level_after);
        # batched execution may reorder independent ops (keyplan/ledger use multisets)
        assert sorted(ev) == sorted(r.events), f"{tag}: trace differs"
        assert len(ev) == len(r.events)
    else:
        # the fast schedule may record MORE rotation events (hoisted rotate-and-sum
        # stages: cheap inner products sharing one ModUp / ModDown) -- only the
        # values and levels must match
        assert any(e[0] == "rotation" for e in ev) == any(e[0] == "rotation" for e in r.events), tag
    return err


def cases(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        W = int(rng.choice([4, 6, 8]))
        C = int(rng.integers(1, 5))
        F = int(rng.integers(1, 5))
        out.append((W, C, F, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("W,C,F,s", cases(9001, 8))
def test_generic_conv(env, W, C, F, s):
    ctx, ref = env
    rng = np.random.default_rng(s)
    while True:
        k = int(rng.choice([2, 3, 5]))
        S = int(rng.integers(1, 4))
        P = int(rng.integers(0, 3))
        if k <= W + 2 * P and (W + 2 * P - k) % S == 0:
            break
    variant = int(rng.integers(0, 2))
    x = rng.uniform(-1, 1, (C, W, W))
    w = rng.uniform(-1, 1, (F, C, k, k))
    b = rng.uniform(-1, 1, F)
    cfg = fh.ConvConfig(C, F, k, S, P, fh.ConvMode.generic, fh.StrideVariant(variant))
    out, ev, r = run_both(ctx, lambda v: fh.convolution(fh.PackedTensor(v, C, W), cfg, fh.KernelTensor(w, b)).data,
                          lambda v: ref.convolution(v, DEPTH, C, W, F, k, S, P, 0, variant, w, b), x)
    check(out, ev, r, f"generic conv W={W} C={C} F={F} k={k} S={S} P={P} v={variant}", ctx.schedule())


@pytest.mark.parametrize("W,C,F,s", cases(9002, 4))
def test_special3x3(env, W, C, F, s):
    ctx, ref = env
    rng = np.random.default_rng(s)
    x = rng.uniform(-1, 1, (C, W, W))
    w = rng.uniform(-1, 1, (F, C, 3, 3))
    b = rng.uniform(-1, 1, F)
    cfg = fh.ConvConfig(C, F, 3, 1, 1, fh.ConvMode.special3x3)
    out, ev, r = run_both(ctx, lambda v: fh.convolution(fh.PackedTensor(v, C, W), cfg, fh.KernelTensor(w, b)).data,
                          lambda v: ref.convolution(v, DEPTH, C, W, F, 3, 1, 1, 1, 0, w, b), x)
    check(out, ev, r, f"special3x3 W={W} C={C} F={F}", ctx.schedule())


@pytest.mark.parametrize("W,C,F,garbage", [(8, 4, 8, True), (16, 8, 16, True), (4, 1, 3, False), (8, 2, 2, True)])
def test_conv2x2_stride2_polyphase(env, W, C, F, garbage):
    """2x2 / stride-2 generic convolution (ResNet-20's downsampling): the fast
    schedule's polyphase path (two masked slot permutations, periodic
    replication, 1x1 channel mixing over the 4C phase blocks)."""
    ctx, ref = env
    rng = np.random.default_rng(W * 1000 + C * 10 + F)
    S = 1 << (LOGN - 1)
    x = np.zeros(S)
    x[:C * W * W] = rng.uniform(-1, 1, C * W * W)
    if garbage:
        x[C * W * W:] = rng.uniform(-1, 1, S - C * W * W)
    w = rng.uniform(-1, 1, (F, C, 2, 2))
    b = rng.uniform(-1, 1, F)
    cfg = fh.ConvConfig(C, F, 2, 2, 0, fh.ConvMode.generic, fh.StrideVariant(0))
    out, ev, r = run_both(ctx, lambda v: fh.convolution(fh.PackedTensor(v, C, W), cfg, fh.KernelTensor(w, b)).data,
                          lambda v: ref.convolution(v, DEPTH, C, W, F, 2, 2, 0, 0, 0, w, b), x)
    check(out, ev, r, f"2x2/s2 conv W={W} C={C} F={F}", ctx.schedule())
    if ctx.schedule() == "fast" and W >= 8:
        assert sum(1 for e in ev if e[0] == "rotation") < sum(1 for e in r.events if e[0] == "rotation")


@pytest.mark.parametrize("W,C,garbage", [(8, 8, False), (4, 16, True), (8, 16, True)])
def test_special3x3_channel_diagonal(env, W, C, garbage):
    """C == F >= 8 with 2 C W^2 <= S: the fast schedule's channel-diagonal
    transform (clean + replicate the input, baby-step/giant-step over channel
    offsets); slots beyond the C blocks carry garbage that must not leak in."""
    ctx, ref = env
    rng = np.random.default_rng(C * 100 + W)
    S = 1 << (LOGN - 1)
    x = np.zeros(S)
    x[:C * W * W] = rng.uniform(-1, 1, C * W * W)
    if garbage:
        x[C * W * W:] = rng.uniform(-1, 1, S - C * W * W)
    w = rng.uniform(-1, 1, (C, C, 3, 3))
    b = rng.uniform(-1, 1, C)
    cfg = fh.ConvConfig(C, C, 3, 1, 1, fh.ConvMode.special3x3)
    out, ev, r = run_both(ctx, lambda v: fh.convolution(fh.PackedTensor(v, C, W), cfg, fh.KernelTensor(w, b)).data,
                          lambda v: ref.convolution(v, DEPTH, C, W, C, 3, 1, 1, 1, 0, w, b), x)
    check(out, ev, r, f"special3x3 diagonal W={W} C={C}", ctx.schedule())
    if ctx.schedule() == "fast":
        assert sum(1 for e in ev if e[0] == "rotation") < sum(1 for e in r.events if e[0] == "rotation")


@pytest.mark.parametrize("W,C,F,s", [c for c in cases(9003, 6) if c[1] >= 2][:3])
def test_grouped_conv(env, W, C, F, s):
    ctx, ref = env
    rng = np.random.default_rng(s)
    Fg = C * int(rng.integers(1, 3))
    while True:
        k = int(rng.choice([2, 3]))
        S = int(rng.integers(1, 3))
        if k <= W and (W - k) % S == 0:
            break
    x = rng.uniform(-1, 1, (C, W, W))
    w = rng.uniform(-1, 1, (Fg, 1, k, k))
    b = rng.uniform(-1, 1, Fg)
    cfg = fh.ConvConfig(C, Fg, k, S, 0, fh.ConvMode.grouped)
    out, ev, r = run_both(ctx, lambda v: fh.convolution(fh.PackedTensor(v, C, W), cfg, fh.KernelTensor(w, b)).data,
                          lambda v: ref.convolution(v, DEPTH, C, W, Fg, k, S, 0, 2, 0, w, b), x)
    check(out, ev, r, f"grouped W={W} C={C} F={Fg} k={k} S={S}", ctx.schedule())


@pytest.mark.parametrize("W,C,F,s", cases(9004, 4))
def test_avg_pool(env, W, C, F, s):
    ctx, ref = env
    rng = np.random.default_rng(s)
    while True:
        k = int(rng.choice([2, 3]))
        S = int(rng.integers(1, 4))
        if k <= W and (W - k) % S == 0:
            break
    variant = int(rng.integers(0, 2))
    x = rng.uniform(-1, 1, (C, W, W))
    cfg = fh.PoolConfig(fh.PoolKind.average, k, S, fh.StrideVariant(variant))
    out, ev, r = run_both(ctx, lambda v: fh.avg_pool(fh.PackedTensor(v, C, W), cfg).data,
                          lambda v: ref.pool(v, DEPTH, C, W, 0, k, S, variant), x)
    check(out, ev, r, f"avg_pool W={W} C={C} k={k} S={S} v={variant}", ctx.schedule())


@pytest.mark.parametrize("W,C,F,s", cases(9005, 3))
def test_global_and_whole_channel_pool(env, W, C, F, s):
    ctx, ref = env
    rng = np.random.default_rng(s)
    x = rng.uniform(-1, 1, (C, W, W))
    out, ev, r = run_both(ctx, lambda v: fh.global_avg_pool(fh.PackedTensor(v, C, W)),
                          lambda v: ref.pool(v, DEPTH, C, W, 1), x)
    check(out, ev, r, f"global W={W} C={C}", ctx.schedule())
    out, ev, r = run_both(ctx, lambda v: fh.whole_channel_pool(fh.PackedTensor(v, C, W), W),
                          lambda v: ref.pool(v, DEPTH, C, W, 2, W), x)
    check(out, ev, r, f"whole_channel W={W} C={C}", ctx.schedule())


@pytest.mark.parametrize("W,C", [(4, 64), (8, 20), (6, 9), (2, 2)])
def test_global_pool_many_channels(env, W, C):
    """Wide channel counts (ResNet-20's 64 x 8 x 8 head): the fast schedule gathers
    the C block heads as one baby-step giant-step slot permutation."""
    ctx, ref = env
    x = np.random.default_rng(9007 + C).uniform(-1, 1, (C, W, W))
    out, ev, r = run_both(ctx, lambda v: fh.global_avg_pool(fh.PackedTensor(v, C, W)),
                          lambda v: ref.pool(v, DEPTH, C, W, 1), x)
    check(out, ev, r, f"global W={W} C={C}", ctx.schedule())
    out, ev, r = run_both(ctx, lambda v: fh.whole_channel_pool(fh.PackedTensor(v, C, W), W),
                          lambda v: ref.pool(v, DEPTH, C, W, 2, W), x)
    check(out, ev, r, f"whole_channel W={W} C={C}", ctx.schedule())


@pytest.mark.parametrize("W,C,F,s", cases(9006, 4))
def test_fully_connected(env, W, C, F, s):
    ctx, ref = env
    rng = np.random.default_rng(s)
    m = int(rng.integers(1, 9))
    B = int(rng.integers(1, 5))
    n = C * W * W
    x = rng.uniform(-1, 1, n)
    w = rng.uniform(-1, 1, (m, n))
    b = rng.uniform(-1, 1, m)
    out, ev, r = run_both(ctx, lambda v: fh.fully_connected(v, fh.FcConfig(n, m, B), fh.FcWeights(w, b)),
                          lambda v: ref.fully_connected(v, DEPTH, n, m, B, w, b), x)
    check(out, ev, r, f"fc n={n} m={m} B={B}", ctx.schedule())


@pytest.mark.parametrize("n,m", [(256, 100), (128, 300), (400, 64)])
def test_fully_connected_wide(env, n, m):
    """Wide FC layers (m >= 64): under the fast schedule the generalised-diagonal
    baby-step giant-step product (layers.cpp fc_diagonal).  Garbage in the input's
    slots beyond n (post-ReLU p(0), say) must be ignored as the reference's row
    products ignore it; output zeros beyond m; same two levels."""
    ctx, ref = env
    rng = np.random.default_rng(n + m)
    S = ctx.slots()
    x = rng.uniform(-1, 1, S)  # n inputs + garbage in [n, S)
    w = rng.uniform(-1, 1, (m, n)) / np.sqrt(n)
    b = rng.uniform(-1, 1, m)
    out, ev, r = run_both(ctx, lambda v: fh.fully_connected(v, fh.FcConfig(n, m, 1), fh.FcWeights(w, b)),
                          lambda v: ref.fully_connected(v, DEPTH, n, m, 1, w, b), x)
    check(out, ev, r, f"fc wide n={n} m={m}", ctx.schedule())
    assert np.abs(out.slots()[m:]).max() < 1e-3


@pytest.mark.parametrize("W,C,F,s", cases(9007, 3))
def test_pad_input(env, W, C, F, s):
    ctx, ref = env
    rng = np.random.default_rng(s)
    P = int(rng.integers(1, 3))
    x = rng.uniform(-1, 1, (C, W, W))
    out, ev, r = run_both(ctx, lambda v: fh.pad_input(fh.PackedTensor(v, C, W), P).data,
                          lambda v: ref.pad_input(v, DEPTH, C, W, P), x)
    check(out, ev, r, f"pad W={W} C={C} P={P}", ctx.schedule())


@pytest.mark.parametrize("W,S,variant", [(4, 2, 0), (8, 2, 1), (8, 3, 0), (6, 2, 1), (8, 4, 1)])
def test_striding(env, W, S, variant):
    ctx, ref = env
    rng = np.random.default_rng(W * 10 + S)
    x = rng.uniform(-1, 1, (1, W, W))
    fn = fh.stride_extract_v2 if variant else fh.stride_extract_v1
    out, ev, r = run_both(ctx, lambda v: fn(v, W, S), lambda v: ref.stride(v, DEPTH, W, S, 0, variant), x)
    check(out, ev, r, f"stride W={W} S={S} v={variant}", ctx.schedule())


@pytest.mark.parametrize("degree,scale", [(7, 1.0), (27, 1.0), (59, 1.0), (59, 8.0)])
def test_secure_relu(env, degree, scale):
    ctx, ref = env
    rng = np.random.default_rng(degree)
    n = 40
    x = rng.uniform(-1, 1, n) * scale
    cfg = fh.ReluConfig(scale, degree, n)
    out, ev, r = run_both(ctx, lambda v: fh.secure_relu(v, cfg), lambda v: ref.secure_relu(v, DEPTH, scale, degree, n),
                          x)
    check(out, ev, r, f"relu degree={degree} scale={scale}", ctx.schedule())


@pytest.mark.parametrize("degree,scale", [(27, 1.0), (59, 8.0)])
def test_secure_relu_many_bit_identical(env, degree, scale):
    """secure_relu_many (the activations of a batch in one polynomial evaluation): per
    input the very words of secure_relu, under both schedules, and the same events thrice."""
    ctx, ref = env
    rng = np.random.default_rng(degree + 1)
    n = 40
    cfg = fh.ReluConfig(scale, degree, n)
    xs = [fh.SlotVector.encode(ctx, rng.uniform(-1, 1, n) * scale) for _ in range(3)]
    rec = ctx.attach_recorder()
    singles = [fh.secure_relu(x, cfg) for x in xs]
    ev1 = sorted((e.kind, e.value) for e in rec.snapshot())
    rec.clear()
    many = fh.secure_relu_many(xs, cfg)
    evm = sorted((e.kind, e.value) for e in rec.snapshot())
    ctx.detach_recorder()
    assert evm == ev1
    for s_, m in zip(singles, many):
        assert m.level() == s_.level()
        assert np.array_equal(m.words(), s_.words())
    assert fh.secure_relu_many([], cfg) == []


@pytest.mark.parametrize("schedule", ["reference", "fast"])
def test_config1_conv_layer(schedule):
    """BASELINE configs[0]: N=2^14, 8192 slots, 50-bit q0 + 40-bit scaling, depth 10, dnum 3;
    1x28x28 U[0,1] input, conv 1->6 5x5 stride 1 pad 0, weights N(0, 0.1^2), bias 0."""
    cfg = fh.ContextConfig.preset("config1")
    cfg.schedule = schedule
    ctx = fh.SlotContext(cfg)
    ref = sref.Ref(16384, 8192, 10)
    rng = np.random.default_rng(1001)
    x = rng.uniform(0, 1, (1, 28, 28))
    w = np.random.default_rng(1002).normal(0, 0.1, (6, 1, 5, 5))
    cfg = fh.ConvConfig(1, 6, 5, 1, 0)
    out, ev, r = run_both(ctx, lambda v: fh.convolution(fh.PackedTensor(v, 1, 28), cfg, fh.KernelTensor(w)).data,
                          lambda v: ref.convolution(v, 10, 1, 28, 6, 5, 1, 0, 0, 0, w, None), x)
    err = check(out, ev, r, "config1 conv", schedule)
    assert r.level == 7 and len(r.rotations()) == 305
    assert err < 1e-4


@pytest.mark.parametrize("W,C,F,k,s,p,mode", [(8, 4, 8, 3, 1, 1, 1), (8, 4, 8, 2, 2, 0, 0), (9, 2, 3, 3, 2, 1, 0),
                                               (9, 2, 3, 3, 2, 0, 0), (12, 1, 6, 5, 1, 0, 0), (8, 3, 4, 3, 1, 1, 0)])
def test_conv_output_clean_past_active(env, W, C, F, k, s, p, mode):
    """Convolutions end in masked placements (layers_conv.cpp:142-177): the slots
    past F * W_out^2 are zero even when the input carries garbage there -- the
    property the model runtime's bootstrap(v, active, clean=True) relies on."""
    ctx, _ = env
    rng = np.random.default_rng(W * 100 + C * 10 + F + k)
    x = rng.uniform(-1, 1, 1 << (LOGN - 1))  # garbage past C * W * W
    w = rng.normal(0, 0.3, (F, C, k, k))
    cfg = fh.ConvConfig(C, F, k, s, p, fh.ConvMode.special3x3 if mode else fh.ConvMode.generic)
    out = fh.convolution(fh.PackedTensor(fh.SlotVector.encode(ctx, x), C, W), cfg, fh.KernelTensor(w)).data
    wo = (W + 2 * p - k) // s + 1
    got = out.slots()
    assert np.abs(got[F * wo * wo:]).max() < 1e-5 * max(1.0, np.abs(got[:F * wo * wo]).max())
