"""GPU: error behaviour of the engine against the reference on the same invalid
inputs.  The reference's errors carry a CLI exit-code category (usage 1, data
2, internal 3; proj/include/slotcnn/errors.hpp:18-80); every case below must
make BOTH the reference (oracle/_ref) and the engine raise, with the same
category and the engine's exception class mirroring the reference's."""
import numpy as np
import pytest

import paper_2510_03996_b200 as fh
from oracle import ref as sref

pytestmark = pytest.mark.gpu

LOGN, DEPTH = 12, 6
N, S = 1 << LOGN, 1 << (LOGN - 1)


@pytest.fixture(scope="module")
def env():
    cfg = fh.ContextConfig(N, S, DEPTH, fh.CryptoMetadata(52, 40, 3), limbs=DEPTH + 1, special_limbs=3,
                           special_bits=60, seed=77, allow_insecure=True)
    return fh.SlotContext(cfg), sref.Ref(N, S, DEPTH)


def both_raise(ours, theirs, cls):
    with pytest.raises(sref.RefError) as r:
        theirs()
    with pytest.raises(fh.Error) as o:
        ours()
    assert isinstance(o.value, cls), f"engine raised {type(o.value).__name__}: {o.value}"
    assert o.value.category == r.value.category, (o.value, r.value)


def vec(n, seed=1):
    return np.random.default_rng(seed).uniform(-1, 1, n)


@pytest.mark.parametrize("t", [S, -S, S + 5])
def test_rotation_out_of_range(env, t):
    ctx, ref = env
    a = vec(S)
    both_raise(lambda: fh.rotate(fh.SlotVector.encode(ctx, a), t),
               lambda: ref.backend_op(0, a, DEPTH, t=t), fh.InvalidRotationError)


def test_mult_plain_at_level_zero(env):
    ctx, ref = env
    a, b = vec(S), vec(S, 2)
    both_raise(lambda: fh.mult_plain(fh.level_down(fh.SlotVector.encode(ctx, a), 1), b),
               lambda: ref.backend_op(3, a, 0, b=b), fh.DepthExhaustedError)


def test_mult_cipher_at_level_zero(env):
    ctx, ref = env
    a, b = vec(S), vec(S, 2)
    both_raise(lambda: fh.mult_cipher(fh.level_down(fh.SlotVector.encode(ctx, a), 1), fh.SlotVector.encode(ctx, b)),
               lambda: ref.backend_op(4, a, 0, b=b, level_b=DEPTH), fh.DepthExhaustedError)


def test_conv_output_exceeds_slots(env):
    ctx, ref = env
    C, W, F, k = 1, 16, 16, 3  # 16 x 14^2 = 3136 > 2048 slots
    x = vec(C * W * W)
    w = vec(F * C * k * k).reshape(F, C, k, k)
    both_raise(lambda: fh.convolution(fh.PackedTensor(fh.SlotVector.encode(ctx, x), C, W),
                                      fh.ConvConfig(C, F, k), fh.KernelTensor(w)),
               lambda: ref.convolution(x, DEPTH, C, W, F, k, 1, 0, 0, 0, w, None), fh.CapacityError)


def test_special3x3_rejects_stride(env):
    ctx, ref = env
    C, W, F = 2, 8, 2
    x = vec(C * W * W)
    w = vec(F * C * 9).reshape(F, C, 3, 3)
    both_raise(lambda: fh.convolution(fh.PackedTensor(fh.SlotVector.encode(ctx, x), C, W),
                                      fh.ConvConfig(C, F, 3, 2, 1, fh.ConvMode.special3x3), fh.KernelTensor(w)),
               lambda: ref.convolution(x, DEPTH, C, W, F, 3, 2, 1, 1, 0, w, None), fh.ShapeError)


@pytest.mark.parametrize("variant", [0, 1])
def test_stride_overruns_input(env, variant):
    ctx, ref = env
    x = vec(64)
    fn = fh.stride_extract_v1 if variant == 0 else fh.stride_extract_v2
    both_raise(lambda: fn(fh.SlotVector.encode(ctx, x), 8, 3, 4),
               lambda: ref.stride(x, DEPTH, 8, 3, 4, variant), fh.ShapeError)


def test_fully_connected_too_wide(env):
    ctx, ref = env
    n, m = S + 1, 2
    w = vec(n * m).reshape(m, n)
    x = vec(S)
    both_raise(lambda: fh.fully_connected(fh.SlotVector.encode(ctx, x), fh.FcConfig(n, m), fh.FcWeights(w)),
               lambda: ref.fully_connected(x, DEPTH, n, m, 1, w), fh.CapacityError)


def test_relu_negative_degree(env):
    ctx, ref = env
    x = vec(40)
    both_raise(lambda: fh.secure_relu(fh.SlotVector.encode(ctx, x), fh.ReluConfig(1.0, -1, 40)),
               lambda: ref.secure_relu(x, DEPTH, 1.0, -1, 40), fh.ShapeError)


def test_relu_out_of_depth(env):
    """degree 59 needs 7 levels; the context has 6."""
    ctx, ref = env
    x = vec(40)
    both_raise(lambda: fh.secure_relu(fh.SlotVector.encode(ctx, x), fh.ReluConfig(1.0, 59, 40)),
               lambda: ref.secure_relu(x, DEPTH, 1.0, 59, 40), fh.DepthExhaustedError)
