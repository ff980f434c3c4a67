"""B200-native RNS-CKKS engine for FHEON's encrypted-CNN hot path.

Host mirror of the reference's backend + layer API (slotcnn) over the C ABI
in include/fheon_b200.h; the compute runs in hand-written sm_100a kernels
(paper_2510_03996_b200/csrc).  See DESIGN.md.
"""
from .api import (  # noqa: F401
    CapacityError, ContextConfig, ConvConfig, ConvMode, CryptoMetadata, CudaError, DepthExhaustedError, Error,
    FcConfig, FcWeights, InternalError, InvalidRotationError, KernelTensor, ModelError, NotImplementedInEngine,
    PackedTensor, PlainVector, PoolConfig, PoolKind, ReluConfig, ShapeError, SlotContext, SlotVector,
    StrideVariant, TraceEvent, TraceRecorder, add, add_plain, avg_pool, bootstrap, bootstrap_many, conv_depth_cost,
    conv_output_width, convolution, flatten, fully_connected, global_avg_pool, host_bootstrap_depth, host_primes,
    host_security, keyswitch_raw,
    level_down,
    mult_cipher, mult_plain, pad_input, rescale, rotate, rotate_hoisted, rotate_many, rotate_sum, rotate_sum_many, secure_relu, secure_relu_many,
    stride_extract_v1,
    stride_extract_v2, sub, unflatten, whole_channel_pool)
from ._native import LIB_PATH, lib  # noqa: F401
