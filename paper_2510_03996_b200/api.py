"""Python mirror of the reference's plugin surface for the hot path.

Names, argument meaning and error behaviour follow slotcnn:
  backend   proj/include/slotcnn/backend.hpp:34-153  (ContextConfig, SlotContext,
            SlotVector, rotate/add/sub/mult_plain/mult_cipher/bootstrap)
  layers    proj/include/slotcnn/layers.hpp:36-158   (ConvConfig, PoolConfig,
            FcConfig, ReluConfig, convolution, avg_pool, ..., *_depth_cost)
  errors    proj/include/slotcnn/errors.hpp:18-80
  trace     proj/include/slotcnn/trace.hpp:22-103
Every call goes through the C ABI into the sm_100a engine; ciphertexts live
in HBM.  PlainVector payloads are host doubles encoded on demand at the
consumer's level and scale.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native


# ---------------------------------------------------------------- errors
class Error(RuntimeError):
    """slotcnn::Error: carries the CLI exit-code category (usage 1, data 2, internal 3)."""

    def __init__(self, message: str, category: int = 3):
        super().__init__(message)
        self.category = category

    @property
    def exit_code(self) -> int:
        return self.category


class InvalidRotationError(Error):
    pass


class DepthExhaustedError(Error):
    pass


class ShapeError(Error):
    pass


class CapacityError(Error):
    pass


class ModelError(Error):
    pass


class InternalError(Error):
    pass


class CudaError(InternalError):
    pass


class NotImplementedInEngine(Error):
    pass


_KIND = {1: InvalidRotationError, 2: DepthExhaustedError, 3: ShapeError, 4: CapacityError, 5: ModelError,
         6: InternalError, 7: CudaError, 8: NotImplementedInEngine}


def _check(rc: int):
    if rc != 0:
        L = _native.lib()
        msg = L.fheon_last_error().decode()
        cls = _KIND.get(L.fheon_last_error_kind(), Error)
        raise cls(msg, rc)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u64ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# ---------------------------------------------------------------- config
@dataclass
class CryptoMetadata:
    """backend.hpp:32-39 -- interpreted here (the reference only carries it)."""
    first_modulus_bits: int = 50
    rescale_bits: int = 40
    key_switch_digits: int = 3
    rescaling_strategy: str = "flexibleauto"


SCHEDULES = {"fast": 0, "reference": 1}


@dataclass
class ContextConfig:
    """backend.hpp:41-59 plus the RNS chain the reference leaves implicit.

    `limbs` defaults to depth_budget + 1 (no bootstrapping: the chain must
    cover the network depth)."""
    ring_dimension: int = 16384
    slot_count: int = 8192
    depth_budget: int = 10
    crypto: CryptoMetadata = field(default_factory=CryptoMetadata)
    limbs: Optional[int] = None
    special_limbs: int = 4
    special_bits: int = 60
    seed: int = 1
    noise_sigma: float = 0.0
    noise_seed: int = 1
    hamming_weight: int = 0   # 0: uniform ternary secret; h: sparse (needed for bootstrapping)
    bootstrap: bool = False   # build the CKKS bootstrapping pipeline
    boot_scale_bits: int = 0  # scale of the bootstrapping levels (0 = rescale_bits)
    digit_split: int = 0      # key-switching digits: 0 uniform, 1 balanced by prime bit size
    # bootstrapping with a dense secret (hamming_weight 0): Hamming weight of the ephemeral
    # sparse secret of the sparse-secret encapsulation (0 = the engine default, 64)
    boot_hamming_weight: int = 0
    # HE-standard security (homomorphicencryption.org 2018, uniform ternary secret): the engine
    # refuses a chain whose log2(QP) exceeds the bound for N at `security` bits, or a sparse
    # main secret, unless allow_insecure (toy rings, the reference's presets) is set
    security: int = 128
    allow_insecure: bool = False
    # a server context without the secret key: evaluation keys arrive by upload
    # (SlotContext.key_upload), encrypt / decrypt are refused
    no_secret: bool = False
    # bootstrapping EvalMod range K (|I| <= K); 0 = the engine default, 16
    boot_k_range: int = 0
    # levels of the bootstrapping linear transforms (0 = 3 each)
    boot_cts_levels: int = 0
    boot_stc_levels: int = 0
    # sparse-slot bootstrapping variants over S/2, ..., S/2^boot_sparse slots (0 = none;
    # bootstrap(v, active_slots) uses them)
    boot_sparse: int = 0
    # layer rotation schedule: "fast" (hoisted / log-depth / baby-step giant-step,
    # same values and levels) or "reference" (the reference's exact rotation trace)
    schedule: str = "fast"

    def validate(self):
        n, s = self.ring_dimension, self.slot_count
        if s <= 0 or s & (s - 1):
            raise ShapeError(f"slot count must be a power of two, got {s}", 2)
        if n <= 0 or n & (n - 1):
            raise ShapeError(f"ring dimension must be a power of two, got {n}", 2)
        if s * 2 != n:
            raise ShapeError(f"slot count {s} must equal half the ring dimension {n} (full packing)", 2)
        if self.schedule not in SCHEDULES:
            raise ShapeError(f'schedule must be one of {sorted(SCHEDULES)}, got "{self.schedule}"', 2)
        if self.depth_budget < 1 and not (self.depth_budget == -1 and self.limbs):
            raise ShapeError(f"depth budget must be positive (or -1 with explicit limbs), got {self.depth_budget}",
                             2)

    @staticmethod
    def preset(name: str) -> "ContextConfig":
        """Named parameter sets.  config1 = BASELINE configs[0] (N=2^14, 50/40-bit,
        depth 10, dnum 3); config2 = configs[1] (N=2^16, L=24 ~50-bit limbs, dnum 3);
        lenet5 / large mirror the reference presets (backend.cpp:61-76).

        Security (he_standard_security): config2 (log2 QP = 1690 <= 1747 at
        N = 2^16) meets 128 bits; config1 (690 > 438 at N = 2^14) and the
        reference's lenet5 / large presets (depth 25 at N = 2^14 / 2^15) cannot,
        so those presets carry allow_insecure=True explicitly."""
        if name == "config1":
            return ContextConfig(16384, 8192, 10, CryptoMetadata(50, 40, 3), limbs=11, special_limbs=4,
                                 special_bits=60, allow_insecure=True)
        if name == "config2":
            return ContextConfig(65536, 32768, 23, CryptoMetadata(60, 50, 3), limbs=24, special_limbs=8,
                                 special_bits=60)
        if name == "lenet5":
            return ContextConfig(16384, 8192, 25, CryptoMetadata(55, 40, 3), limbs=26, special_limbs=9,
                                 special_bits=60, allow_insecure=True)
        if name == "large":
            return ContextConfig(32768, 16384, 25, CryptoMetadata(55, 40, 3), limbs=26, special_limbs=9,
                                 special_bits=60, allow_insecure=True)
        raise ModelError(f'unknown context preset "{name}"', 2)

    def params(self) -> _native.fheon_params:
        self.validate()
        L = self.limbs if self.limbs is not None else self.depth_budget + 1
        p = _native.fheon_params()
        p.log_n = int(self.ring_dimension).bit_length() - 1
        p.limbs = L
        p.special_limbs = self.special_limbs
        p.dnum = self.crypto.key_switch_digits
        p.first_mod_bits = self.crypto.first_modulus_bits
        p.scale_bits = self.crypto.rescale_bits
        p.special_bits = self.special_bits
        p.depth_budget = self.depth_budget
        p.seed = self.seed
        p.hamming_weight = self.hamming_weight
        p.bootstrap = int(bool(self.bootstrap))
        p.boot_scale_bits = int(self.boot_scale_bits)
        p.digit_split = int(self.digit_split)
        p.boot_hamming_weight = int(self.boot_hamming_weight)
        p.min_security = int(self.security)
        p.allow_insecure = int(bool(self.allow_insecure))
        p.no_secret = int(bool(self.no_secret))
        p.boot_k_range = int(self.boot_k_range)
        p.boot_cts_levels = int(self.boot_cts_levels)
        p.boot_stc_levels = int(self.boot_stc_levels)
        p.boot_sparse = int(self.boot_sparse)
        return p


@dataclass
class TraceEvent:
    kind: str  # "rotation" | "mult_plain" | "mult_cipher" | "bootstrap"
    value: int


_TRACE_KIND = {0: "rotation", 1: "mult_plain", 2: "mult_cipher", 3: "bootstrap"}


class TraceRecorder:
    """View over the engine's trace (trace.hpp:37-103)."""

    def __init__(self, ctx: "SlotContext"):
        self._ctx = ctx

    def snapshot(self) -> List[TraceEvent]:
        L = _native.lib()
        n = C.c_size_t()
        _check(L.fheon_trace(self._ctx._h, None, 0, C.byref(n)))
        buf = (C.c_long * (2 * max(1, n.value)))()
        _check(L.fheon_trace(self._ctx._h, buf, n.value, C.byref(n)))
        return [TraceEvent(_TRACE_KIND[buf[2 * i]], buf[2 * i + 1]) for i in range(n.value)]

    def rotation_indices(self) -> List[int]:
        return [e.value for e in self.snapshot() if e.kind == "rotation"]

    def rotation_usage(self) -> Dict[int, int]:
        out: Dict[int, int] = {}
        for t in self.rotation_indices():
            out[t] = out.get(t, 0) + 1
        return dict(sorted(out.items()))

    def clear(self):
        _check(_native.lib().fheon_trace_clear(self._ctx._h))


class SlotContext:
    """SlotContext::create (backend.hpp:66-93): owns the device context."""

    def __init__(self, config: ContextConfig, _share_keys_from: Optional["SlotContext"] = None):
        self.config = config
        L = _native.lib()
        p = config.params()
        h = C.c_void_p()
        if _share_keys_from is None:
            _check(L.fheon_ctx_create(C.byref(p), C.byref(h)))
        else:
            _check(L.fheon_ctx_clone(_share_keys_from._h, C.byref(h)))
        self._h = h
        self.L = p.limbs
        self.K = p.special_limbs
        self.dnum = p.dnum
        self.N = config.ring_dimension
        self._recorder: Optional[TraceRecorder] = None
        primes = np.zeros(self.L + self.K, np.uint64)
        scales = np.zeros(self.L, np.float64)
        slots = C.c_int()
        _check(L.fheon_ctx_info(h, _u64ptr(primes), _dptr(scales), C.byref(slots)))
        self.primes = primes
        self.scales = scales
        self._slots = slots.value
        _check(L.fheon_ctx_set_schedule(h, SCHEDULES[config.schedule]))

    @staticmethod
    def create(config: ContextConfig) -> "SlotContext":
        return SlotContext(config)

    def clone(self) -> "SlotContext":
        """A second context (own CUDA stream, pools, caches) over the same parameters and
        secret that shares this one's resident evaluation keys: several images in flight
        on one GPU, one host thread per context, without duplicating the keys."""
        return SlotContext(self.config, _share_keys_from=self)

    def __del__(self):
        self.close()

    def close(self):
        """Destroy the engine context now (keys, pools, caches) instead of at garbage
        collection; ciphertexts of this context must not be used afterwards."""
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().fheon_ctx_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def slots(self) -> int:
        return self._slots

    def security(self) -> Dict[str, object]:
        """log2(QP), ring dimension and the HE-standard security level of the chain."""
        lq, lev = C.c_double(), C.c_int()
        _check(_native.lib().fheon_ctx_security(self._h, C.byref(lq), C.byref(lev)))
        return security_report(self.N, lq.value, lev.value, self.config)

    def depth_budget(self) -> int:
        """Levels of fresh encryptions and bootstrap outputs (resolved by the engine)."""
        return int(_native.lib().fheon_ctx_depth_budget(self._h))

    def schedule(self) -> str:
        v = int(_native.lib().fheon_ctx_schedule(self._h))
        return {k: n for n, k in SCHEDULES.items()}[v]

    def set_schedule(self, schedule: str):
        if schedule not in SCHEDULES:
            raise ShapeError(f'schedule must be one of {sorted(SCHEDULES)}, got "{schedule}"', 2)
        _check(_native.lib().fheon_ctx_set_schedule(self._h, SCHEDULES[schedule]))

    def packed_words(self, limbs: int) -> int:
        """uint64 words of one ciphertext with `limbs` limbs in the packed wire format."""
        n = int(_native.lib().fheon_ct_packed_words(self._h, int(limbs)))
        if n == 0:
            raise ShapeError(f"bad limb count {limbs}", 2)
        return n

    def wait_transfers(self):
        """Block until every asynchronous upload / download has completed."""
        _check(_native.lib().fheon_ctx_wait_transfers(self._h))
        self._keep = []

    def set_weight_cache(self, nbytes: int):
        """HBM budget of resident weight plaintexts (weight_mode "preload"); 0 = "lazy"."""
        _check(_native.lib().fheon_ctx_set_weight_cache(self._h, int(nbytes)))

    def attach_recorder(self) -> TraceRecorder:
        _check(_native.lib().fheon_set_tracing(self._h, 1))
        _check(_native.lib().fheon_trace_clear(self._h))
        self._recorder = TraceRecorder(self)
        return self._recorder

    def detach_recorder(self):
        _check(_native.lib().fheon_set_tracing(self._h, 0))
        self._recorder = None

    def recorder(self) -> Optional[TraceRecorder]:
        return self._recorder

    # ---- keys
    def galois_element(self, t: int) -> int:
        return int(_native.lib().fheon_galois_elt(self._h, int(t)))

    def keygen_rotations(self, steps: Sequence[int]):
        arr = (C.c_long * max(1, len(steps)))(*[int(s) for s in steps])
        _check(_native.lib().fheon_keygen_rotations(self._h, arr, len(steps)))

    def keygen_relin(self):
        _check(_native.lib().fheon_keygen_relin(self._h))

    def set_strict_keys(self, strict: bool):
        _check(_native.lib().fheon_set_strict_keys(self._h, int(bool(strict))))

    def key_bytes(self) -> int:
        """HBM bytes of the resident evaluation keys."""
        return int(_native.lib().fheon_key_bytes(self._h))

    def prefetch_rotation_keys(self, steps: Sequence[int]):
        """Generate the rotation keys of `steps` now (stream-ordered, no host sync)."""
        arr = (C.c_long * max(1, len(steps)))(*[int(s) for s in steps])
        _check(_native.lib().fheon_prefetch_rotation_keys(self._h, arr, len(steps)))

    def drop_rotation_keys(self, steps: Sequence[int]):
        """Evict the rotation keys of `steps` (regenerated bit-identically on demand)."""
        arr = (C.c_long * max(1, len(steps)))(*[int(s) for s in steps])
        _check(_native.lib().fheon_drop_rotation_keys(self._h, arr, len(steps)))

    def key_events(self) -> Dict[str, int]:
        g, d = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        _check(_native.lib().fheon_key_events(self._h, _u64ptr(g), _u64ptr(d)))
        return {"generated": int(g[0]), "dropped": int(d[0])}

    def key_count(self) -> int:
        return int(_native.lib().fheon_key_count(self._h))

    def download_key(self, key_id: int) -> np.ndarray:
        out = np.zeros((self.dnum, 2, self.L + self.K, self.N), np.uint64)
        _check(_native.lib().fheon_key_download(self._h, key_id, _u64ptr(out)))
        return out

    # ---- misc
    # ---- evaluation-key serialization / upload (client -> server, keyplan streaming)
    def key_packed_words(self) -> int:
        return int(_native.lib().fheon_key_packed_words(self._h))

    def key_download_packed(self, key_id: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """The key's packed wire-format words (standard form, every limb at its prime's bit width)."""
        if out is None:
            out = np.zeros(self.key_packed_words(), np.uint64)
        _check(_native.lib().fheon_key_download_packed(self._h, int(key_id), _u64ptr(out)))
        return out

    def key_upload(self, key_id: int, words: np.ndarray, packed: bool = True, async_copy: bool = False):
        """Make an evaluation key resident from host words (packed wire format, or raw
        [dnum][2][L+K][N] standard form).  async_copy: on the upload stream (keep the
        pinned host buffer alive until wait_transfers)."""
        w = np.ascontiguousarray(words, np.uint64)
        if async_copy:
            if not packed:
                raise ShapeError("asynchronous key upload takes the packed format", 2)
            self._keep = getattr(self, "_keep", [])
            self._keep.append(w)
            _check(_native.lib().fheon_key_upload_packed_async(self._h, int(key_id), _u64ptr(w)))
        elif packed:
            _check(_native.lib().fheon_key_upload_packed(self._h, int(key_id), _u64ptr(w)))
        else:
            _check(_native.lib().fheon_key_upload(self._h, int(key_id), _u64ptr(w)))

    def required_key_ids(self) -> List[int]:
        """Relinearisation, conjugation, bootstrapping rotations and encapsulation keys
        the context needs beyond rotation keys (what a client uploads to a server)."""
        n = C.c_size_t()
        _check(_native.lib().fheon_required_key_ids(self._h, None, 0, C.byref(n)))
        ids = np.zeros(n.value, np.uint64)
        _check(_native.lib().fheon_required_key_ids(self._h, _u64ptr(ids), n.value, C.byref(n)))
        return [int(i) for i in ids]

    def key_uploads(self) -> Dict[str, int]:
        c, b = C.c_uint64(), C.c_uint64()
        _check(_native.lib().fheon_key_uploads(self._h, C.byref(c), C.byref(b)))
        return {"uploads": c.value, "bytes": b.value}

    def stream(self) -> int:
        return int(_native.lib().fheon_ctx_stream(self._h) or 0)

    def sync(self):
        _check(_native.lib().fheon_ctx_sync(self._h))

    def stats(self) -> Dict[str, int]:
        a = np.zeros(9, np.uint64)
        _check(_native.lib().fheon_ctx_stats(self._h, _u64ptr(a)))
        keys = ["rotations", "keyswitches", "mult_plain", "mult_cipher", "rescales", "ntt_limbs", "encodes", "adds",
                "launches"]
        return {k: int(v) for k, v in zip(keys, a)}

    def reset_stats(self):
        _check(_native.lib().fheon_ctx_reset_stats(self._h))

    def timer_arm(self, kernel_class: int):
        _check(_native.lib().fheon_timer_arm(self._h, int(kernel_class)))

    def timer_read(self):
        ms, n = C.c_double(), C.c_int()
        _check(_native.lib().fheon_timer_read(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def microbench(self, kind: int, batch: int, limbs: int, n_rot: int = 1, iters: int = 10) -> float:
        ms = C.c_double()
        _check(_native.lib().fheon_microbench(self._h, kind, batch, limbs, n_rot, iters, C.byref(ms)))
        return ms.value

    # ---- raw RNS primitives (parity tests)
    def ntt(self, words: np.ndarray, inverse: bool = False) -> np.ndarray:
        a = np.ascontiguousarray(words, np.uint64).copy()
        if a.ndim == 2:
            npolys, nl = 1, a.shape[0]
        else:
            npolys, nl = a.shape[0], a.shape[1]
        _check(_native.lib().fheon_ntt_host(self._h, _u64ptr(a), npolys, nl, int(inverse)))
        return a

    def automorph(self, words: np.ndarray, g: int) -> np.ndarray:
        a = np.ascontiguousarray(words, np.uint64).copy()
        if a.ndim == 2:
            npolys, nl = 1, a.shape[0]
        else:
            npolys, nl = a.shape[0], a.shape[1]
        _check(_native.lib().fheon_automorph_host(self._h, _u64ptr(a), npolys, nl, g))
        return a


class SlotVector:
    """Device ciphertext handle (SlotVector, backend.hpp:108-132)."""

    def __init__(self, ctx: SlotContext, handle):
        self._ctx = ctx
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().fheon_ct_free(h)
            except Exception:  # interpreter shutdown: module state already torn down
                pass
            self._h = None

    @staticmethod
    def encode(ctx: SlotContext, values: Sequence[float]) -> "SlotVector":
        """SlotVector::encode (backend.cpp:148-161): encrypt at the depth budget."""
        v = np.ascontiguousarray(values, np.float64)
        h = C.c_void_p()
        _check(_native.lib().fheon_encrypt(ctx._h, _dptr(v), v.size, C.byref(h)))
        return SlotVector(ctx, h)

    @staticmethod
    def encode_top(ctx: SlotContext, values: Sequence[float]) -> "SlotVector":
        v = np.ascontiguousarray(values, np.float64)
        h = C.c_void_p()
        _check(_native.lib().fheon_encrypt_top(ctx._h, _dptr(v), v.size, C.byref(h)))
        return SlotVector(ctx, h)

    @staticmethod
    def from_words(ctx: SlotContext, words: np.ndarray, scale: float, async_copy: bool = False) -> "SlotVector":
        """Upload raw RNS words [2][limbs][N].  async_copy: non-blocking copy on the
        context's upload stream -- `words` must be a contiguous uint64 array (pinned
        for overlap) that stays valid until SlotContext.wait_transfers()."""
        if async_copy:
            if words.dtype != np.uint64 or not words.flags.c_contiguous:
                raise ShapeError("async upload needs a contiguous uint64 array", 2)
            w = words
        else:
            w = np.ascontiguousarray(words, np.uint64)
        h = C.c_void_p()
        fn = _native.lib().fheon_ct_upload_async if async_copy else _native.lib().fheon_ct_upload
        _check(fn(ctx._h, _u64ptr(w), w.shape[1], float(scale), C.byref(h)))
        return SlotVector(ctx, h)

    @staticmethod
    def from_packed(ctx: SlotContext, packed: np.ndarray, limbs: int, scale: float,
                    async_copy: bool = False) -> "SlotVector":
        """Upload a ciphertext in the packed wire format (include/fheon_b200.h:
        fheon_ct_upload_packed): ctx.packed_words(limbs) uint64 words, unpacked on
        the device.  async_copy as for from_words."""
        want = ctx.packed_words(limbs)
        if packed.dtype != np.uint64 or not packed.flags.c_contiguous or packed.size != want:
            raise ShapeError(f"packed ciphertext must be {want} contiguous uint64 words", 2)
        h = C.c_void_p()
        fn = _native.lib().fheon_ct_upload_packed_async if async_copy else _native.lib().fheon_ct_upload_packed
        _check(fn(ctx._h, _u64ptr(packed), int(limbs), float(scale), C.byref(h)))
        return SlotVector(ctx, h)

    def packed(self, out: Optional[np.ndarray] = None, async_copy: bool = False) -> np.ndarray:
        """Download in the packed wire format (packed on the device)."""
        want = self._ctx.packed_words(self.limbs())
        if out is None:
            if async_copy:
                raise ShapeError("async download needs a caller-owned output buffer", 2)
            out = np.zeros(want, np.uint64)
        elif out.size != want or out.dtype != np.uint64 or not out.flags.c_contiguous:
            raise ShapeError(f"output buffer must be {want} contiguous uint64 words", 2)
        fn = _native.lib().fheon_ct_download_packed_async if async_copy else _native.lib().fheon_ct_download_packed
        _check(fn(self._ctx._h, self._h, _u64ptr(out)))
        return out

    def valid(self) -> bool:
        return bool(self._h)

    def context(self) -> SlotContext:
        return self._ctx

    def level(self) -> int:
        return int(_native.lib().fheon_ct_level(self._h))

    def limbs(self) -> int:
        return int(_native.lib().fheon_ct_limbs(self._h))

    def scale(self) -> float:
        return float(_native.lib().fheon_ct_scale(self._h))

    def size(self) -> int:
        return self._ctx.slots()

    def slots(self) -> np.ndarray:
        """Decrypt + decode (client side)."""
        out = np.zeros(self._ctx.slots(), np.float64)
        _check(_native.lib().fheon_decrypt(self._ctx._h, self._h, _dptr(out), out.size))
        return out

    def slots_complex(self) -> np.ndarray:
        re = np.zeros(self._ctx.slots(), np.float64)
        im = np.zeros(self._ctx.slots(), np.float64)
        _check(_native.lib().fheon_decrypt_complex(self._ctx._h, self._h, _dptr(re), _dptr(im), re.size))
        return re + 1j * im

    def words(self, out: Optional[np.ndarray] = None, async_copy: bool = False) -> np.ndarray:
        """Download raw RNS words.  async_copy: returns at once; `out` is filled on the
        context's download stream and is valid after SlotContext.wait_transfers()."""
        shape = (2, self.limbs(), self._ctx.N)
        if out is None:
            if async_copy:
                raise ShapeError("async download needs a caller-owned output buffer", 2)
            out = np.zeros(shape, np.uint64)
        elif out.shape != shape or out.dtype != np.uint64 or not out.flags.c_contiguous:
            raise ShapeError(f"output buffer must be a contiguous uint64 array of shape {shape}", 2)
        fn = _native.lib().fheon_ct_download_async if async_copy else _native.lib().fheon_ct_download
        _check(fn(self._ctx._h, self._h, _u64ptr(out)))
        return out


def _wrap(ctx, fn, *args) -> SlotVector:
    h = C.c_void_p()
    _check(fn(ctx._h, *args, C.byref(h)))
    return SlotVector(ctx, h)


def _vec(ctx: SlotContext, p) -> np.ndarray:
    v = np.ascontiguousarray(getattr(p, "slots", p), np.float64)
    return v


# ---------------------------------------------------------------- backend ops
@dataclass
class PlainVector:
    slots: np.ndarray

    @staticmethod
    def zeros(n: int) -> "PlainVector":
        return PlainVector(np.zeros(n))

    @staticmethod
    def from_values(n: int, values: Sequence[float]) -> "PlainVector":
        values = np.asarray(values, np.float64)
        if values.size > n:
            raise CapacityError(f"plain vector payload of {values.size} values does not fit in {n} slots", 2)
        out = np.zeros(n)
        out[: values.size] = values
        return PlainVector(out)


def rotate(v: SlotVector, t: int) -> SlotVector:
    return _wrap(v._ctx, _native.lib().fheon_rotate, v._h, int(t))


def rotate_hoisted(v: SlotVector, ts: Sequence[int]) -> List[SlotVector]:
    n = len(ts)
    arr = (C.c_long * max(1, n))(*[int(t) for t in ts])
    outs = (C.c_void_p * max(1, n))()
    _check(_native.lib().fheon_rotate_hoisted(v._ctx._h, v._h, arr, n, outs))
    return [SlotVector(v._ctx, C.c_void_p(outs[i])) for i in range(n)]


def rotate_many(xs: Sequence[SlotVector], ts: Sequence[int]) -> List[SlotVector]:
    """xs[i] rotated by ts[i] in one batched key-switch pipeline."""
    n = len(xs)
    if n != len(ts):
        raise ShapeError("rotate_many: xs and ts differ in length", 2)
    if n == 0:
        return []
    ctx = xs[0]._ctx
    hs = (C.c_void_p * n)(*[x._h.value if isinstance(x._h, C.c_void_p) else x._h for x in xs])
    arr = (C.c_long * n)(*[int(t) for t in ts])
    outs = (C.c_void_p * n)()
    _check(_native.lib().fheon_rotate_many(ctx._h, hs, arr, n, outs))
    return [SlotVector(ctx, C.c_void_p(outs[i])) for i in range(n)]


def rotate_sum_many(groups: Sequence[Sequence[Tuple[SlotVector, int]]]) -> List[SlotVector]:
    """[sum_k rotate(x_rk, t_rk) for every group r] in one key-switch pipeline."""
    flat = [p for g in groups for p in g]
    if not groups or any(len(g) == 0 for g in groups):
        raise ShapeError("rotate_sum_many: every group needs at least one term", 2)
    ctx = flat[0][0]._ctx
    n = len(flat)
    hs = (C.c_void_p * n)(*[x._h.value if isinstance(x._h, C.c_void_p) else x._h for x, _ in flat])
    arr = (C.c_long * n)(*[int(t) for _, t in flat])
    sizes = (C.c_size_t * len(groups))(*[len(g) for g in groups])
    outs = (C.c_void_p * len(groups))()
    _check(_native.lib().fheon_rotate_sum_many(ctx._h, hs, arr, sizes, len(groups), outs))
    return [SlotVector(ctx, C.c_void_p(o)) for o in outs]


def rotate_sum(xs: Sequence[SlotVector], ts: Sequence[int]) -> SlotVector:
    """sum_i rotate(xs[i], ts[i]) with one ModDown (rotate-and-sum key switch)."""
    n = len(xs)
    if n != len(ts) or n == 0:
        raise ShapeError("rotate_sum: xs and ts must be non-empty and of equal length", 2)
    ctx = xs[0]._ctx
    hs = (C.c_void_p * n)(*[x._h.value if isinstance(x._h, C.c_void_p) else x._h for x in xs])
    arr = (C.c_long * n)(*[int(t) for t in ts])
    out = (C.c_void_p * 1)()
    _check(_native.lib().fheon_rotate_sum(ctx._h, hs, arr, n, out))
    return SlotVector(ctx, C.c_void_p(out[0]))


def add(a: SlotVector, b: SlotVector) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_add, a._h, b._h)


def sub(a: SlotVector, b: SlotVector) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_sub, a._h, b._h)


def add_plain(a: SlotVector, p) -> SlotVector:
    v = _vec(a._ctx, p)
    return _wrap(a._ctx, _native.lib().fheon_add_plain, a._h, _dptr(v), v.size)


def mult_plain(a: SlotVector, p) -> SlotVector:
    v = _vec(a._ctx, p)
    return _wrap(a._ctx, _native.lib().fheon_mult_plain, a._h, _dptr(v), v.size)


def mult_cipher(a: SlotVector, b: SlotVector) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_mult_cipher, a._h, b._h)


def bootstrap(a: SlotVector, active_slots: Optional[int] = None, clean: bool = False) -> SlotVector:
    """backend.cpp:233-249: refresh to the depth budget.  With `active_slots`, only
    slots [0, active_slots) are kept (a sparse-slot variant when the context has
    one that fits and the input sits above level 0 -- or at any level when `clean`:
    the caller asserts slots past active_slots are zero; the rest become 0)."""
    if active_slots is None:
        return _wrap(a._ctx, _native.lib().fheon_bootstrap, a._h)
    return _wrap(a._ctx, _native.lib().fheon_bootstrap_active, a._h, int(active_slots), int(bool(clean)))


def bootstrap_many(xs: Sequence[SlotVector], active_slots: int, clean: bool = False) -> List[SlotVector]:
    """bootstrap(x, active_slots, clean) of every x in lockstep (the images of a
    batched inference): inputs on one level share each stage's launches, so keys and
    encoded diagonals leave HBM once per batch.  Bit-identical to the single calls."""
    n = len(xs)
    if n == 0:
        return []
    ctx = xs[0]._ctx
    hs = (C.c_void_p * n)(*[x._h.value if isinstance(x._h, C.c_void_p) else x._h for x in xs])
    outs = (C.c_void_p * n)()
    _check(_native.lib().fheon_bootstrap_active_many(ctx._h, hs, n, int(active_slots), int(bool(clean)), outs))
    return [SlotVector(ctx, C.c_void_p(outs[i])) for i in range(n)]


def bootstrap_stage(a: SlotVector, stage: int) -> SlotVector:
    """Bootstrapping stage probe: 1 CoeffsToSlots, 2 EvalMod, 3 SlotsToCoeffs, 4 ModRaise."""
    return _wrap(a._ctx, _native.lib().fheon_bootstrap_stage, a._h, int(stage))


def bootstrap_info(ctx: "SlotContext"):
    info = (C.c_int * 4)()
    n = C.c_size_t()
    _check(_native.lib().fheon_bootstrap_info(ctx._h, info, None, 0, C.byref(n)))
    coeffs = np.zeros(n.value)
    _check(_native.lib().fheon_bootstrap_info(ctx._h, info, _dptr(coeffs), n.value, C.byref(n)))
    return {"depth": info[0], "k_range": info[1], "double_angles": info[2], "stc_input_limbs": info[3],
            "cos_coeffs": coeffs}


def rescale(a: SlotVector) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_rescale, a._h)


def level_down(a: SlotVector, limbs: int) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_level_down, a._h, int(limbs))


def keyswitch_raw(a: SlotVector, key_id: int, g: int) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_keyswitch_raw, a._h, int(key_id), int(g))


# ---------------------------------------------------------------- layers
class ConvMode(IntEnum):
    generic = 0
    special3x3 = 1
    grouped = 2


class StrideVariant(IntEnum):
    extract = 0
    masked = 1


class PoolKind(IntEnum):
    average = 0
    global_ = 1
    whole_channel = 2


@dataclass
class ConvConfig:
    in_channels: int = 1
    out_channels: int = 1
    kernel: int = 1
    stride: int = 1
    padding: int = 0
    mode: ConvMode = ConvMode.generic
    stride_variant: StrideVariant = StrideVariant.extract

    def c(self) -> _native.fheon_conv_cfg:
        return _native.fheon_conv_cfg(self.in_channels, self.out_channels, self.kernel, self.stride, self.padding,
                                      int(self.mode), int(self.stride_variant))


@dataclass
class PoolConfig:
    kind: PoolKind = PoolKind.average
    kernel: int = 2
    stride: int = 2
    stride_variant: StrideVariant = StrideVariant.extract


@dataclass
class FcConfig:
    inputs: int = 0
    outputs: int = 0
    merge_budget: int = 1


@dataclass
class ReluConfig:
    scale: float = 1.0
    degree: int = 59
    active_slots: int = 0


@dataclass
class KernelTensor:
    """(F, C, k, k) weights + bias (tensors.hpp:40-76)."""
    weights: np.ndarray
    bias: Optional[np.ndarray] = None

    @property
    def out_channels(self):
        return self.weights.shape[0]


@dataclass
class FcWeights:
    weights: np.ndarray  # (m, n)
    bias: Optional[np.ndarray] = None


@dataclass
class PackedTensor:
    data: SlotVector
    channels: int
    width: int

    def used_slots(self) -> int:
        return self.channels * self.width * self.width


def flatten(ctx: SlotContext, t: np.ndarray) -> PackedTensor:
    """packing.cpp:10-28: (C, W, W) host tensor -> channel-major slots, encrypted."""
    t = np.asarray(t, np.float64)
    if t.ndim != 3 or t.shape[1] != t.shape[2]:
        raise ShapeError(f"packed tensors must be square (C, W, W); got {t.shape}", 2)
    if t.size > ctx.slots():
        raise CapacityError(f"tensor needs {t.size} slots but the context provides {ctx.slots()}", 2)
    return PackedTensor(SlotVector.encode(ctx, t.reshape(-1)), t.shape[0], t.shape[1])


def unflatten(p: PackedTensor) -> np.ndarray:
    s = p.data.slots()
    return s[: p.used_slots()].reshape(p.channels, p.width, p.width)


def conv_output_width(W: int, k: int, S: int, P: int) -> int:
    if k == 0 or S == 0:
        raise ShapeError("kernel and stride must be positive", 2)
    Wp = W + 2 * P
    if k > Wp:
        raise ShapeError(f"kernel edge {k} exceeds padded input edge {Wp}", 2)
    if (Wp - k) % S != 0:
        raise ShapeError(f"geometry is not divisible: ({Wp} - {k}) is not a multiple of stride {S}", 2)
    return (Wp - k) // S + 1


def convolution(x: PackedTensor, cfg: ConvConfig, w: KernelTensor) -> PackedTensor:
    ctx = x.data._ctx
    wt = np.ascontiguousarray(w.weights, np.float64)
    b = None if w.bias is None else np.ascontiguousarray(w.bias, np.float64)
    c = cfg.c()
    h = C.c_void_p()
    oc, ow = C.c_size_t(), C.c_size_t()
    _check(_native.lib().fheon_convolution(ctx._h, x.data._h, x.channels, x.width, C.byref(c), _dptr(wt),
                                           _dptr(b) if b is not None else None, C.byref(h), C.byref(oc),
                                           C.byref(ow)))
    return PackedTensor(SlotVector(ctx, h), oc.value, ow.value)


def _pool(x: PackedTensor, kind, k, s, variant):
    ctx = x.data._ctx
    h = C.c_void_p()
    oc, ow = C.c_size_t(), C.c_size_t()
    _check(_native.lib().fheon_pool(ctx._h, x.data._h, x.channels, x.width, int(kind), k, s, int(variant),
                                    C.byref(h), C.byref(oc), C.byref(ow)))
    return SlotVector(ctx, h), oc.value, ow.value


def avg_pool(x: PackedTensor, cfg: PoolConfig) -> PackedTensor:
    if cfg.kind != PoolKind.average:
        raise ShapeError("avg_pool handles the windowed average kind only", 2)
    v, c, w = _pool(x, 0, cfg.kernel, cfg.stride, cfg.stride_variant)
    return PackedTensor(v, c, w)


def global_avg_pool(x: PackedTensor) -> SlotVector:
    return _pool(x, 1, 0, 0, 0)[0]


def whole_channel_pool(x: PackedTensor, k: int) -> SlotVector:
    return _pool(x, 2, k, 0, 0)[0]


def fully_connected(x, cfg: FcConfig, w: FcWeights) -> SlotVector:
    if isinstance(x, PackedTensor):
        if cfg.inputs != x.used_slots():
            raise ShapeError(f"fully-connected layer expects {cfg.inputs} inputs, packed tensor provides "
                             f"{x.used_slots()}", 2)
        x = x.data
    wt = np.ascontiguousarray(w.weights, np.float64)
    if wt.shape != (cfg.outputs, cfg.inputs):
        raise ShapeError(f"weight matrix is {wt.shape[0]}x{wt.shape[1]}, layer expects "
                         f"{cfg.outputs}x{cfg.inputs}", 2)
    b = None if w.bias is None else np.ascontiguousarray(w.bias, np.float64)
    return _wrap(x._ctx, _native.lib().fheon_fully_connected, x._h, cfg.inputs, cfg.outputs, cfg.merge_budget,
                 _dptr(wt), _dptr(b) if b is not None else None)


def secure_relu(x, cfg: ReluConfig):
    if isinstance(x, PackedTensor):
        active = cfg.active_slots or x.used_slots()
        v = _wrap(x.data._ctx, _native.lib().fheon_secure_relu, x.data._h, float(cfg.scale), int(cfg.degree),
                  int(active))
        return PackedTensor(v, x.channels, x.width)
    return _wrap(x._ctx, _native.lib().fheon_secure_relu, x._h, float(cfg.scale), int(cfg.degree),
                 int(cfg.active_slots))


def secure_relu_many(xs: Sequence[SlotVector], cfg: ReluConfig) -> List[SlotVector]:
    """secure_relu(x, cfg) of every x in lockstep (one polynomial evaluation carrying
    the whole batch); bit-identical to the single calls."""
    n = len(xs)
    if n == 0:
        return []
    ctx = xs[0]._ctx
    hs = (C.c_void_p * n)(*[x._h.value if isinstance(x._h, C.c_void_p) else x._h for x in xs])
    outs = (C.c_void_p * n)()
    _check(_native.lib().fheon_secure_relu_many(ctx._h, hs, n, float(cfg.scale), int(cfg.degree),
                                                int(cfg.active_slots), outs))
    return [SlotVector(ctx, C.c_void_p(outs[i])) for i in range(n)]


def stride_extract_v1(a: SlotVector, W: int, S: int, W_out: int = 0) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_stride, a._h, W, S, W_out, 0)


def stride_extract_v2(a: SlotVector, W: int, S: int, W_out: int = 0) -> SlotVector:
    return _wrap(a._ctx, _native.lib().fheon_stride, a._h, W, S, W_out, 1)


def pad_input(x: PackedTensor, padding: int) -> PackedTensor:
    if padding == 0:
        return x
    v = _wrap(x.data._ctx, _native.lib().fheon_pad_input, x.data._h, x.channels, x.width, padding)
    return PackedTensor(v, x.channels, x.width + 2 * padding)


def host_primes(config: ContextConfig):
    """Prime chain and per-level scale targets, computed on the host (no GPU needed)."""
    p = config.params()
    primes = np.zeros(p.limbs + p.special_limbs, np.uint64)
    scales = np.zeros(p.limbs, np.float64)
    _check(_native.lib().fheon_host_primes(C.byref(p), _u64ptr(primes), _dptr(scales)))
    return primes, scales


def security_report(N: int, log_qp: float, level: int, config: ContextConfig) -> Dict[str, object]:
    sparse = config.hamming_weight > 0
    return {"ring_dimension": int(N), "log2_qp": round(float(log_qp), 1),
            "he_standard_128_bound": {1 << 14: 438, 1 << 15: 881, 1 << 16: 1747}.get(int(N)),
            "security_bits": None if level < 0 else int(level),
            "meets_128": bool(level >= 128),
            "secret": (f"sparse ternary h={config.hamming_weight} (not covered by the HE-standard table)" if sparse
                       else "uniform ternary" + (f"; bootstrapping via sparse-secret encapsulation (ephemeral h="
                                                 f"{config.boot_hamming_weight or 64} on q_0 and P only, EvalMod "
                                                 f"range {config.boot_k_range or 16})"
                                                 if config.bootstrap else "")),
            "estimate": "HE standard (homomorphicencryption.org 2018) Table 1, uniform ternary, classical; "
                        "N = 2^16 row as shipped by OpenFHE (1747 / 1224 / 956 bits)"}


def release_memory():
    """Synchronise and return the engine pool's unused device memory (between workloads)."""
    import gc
    gc.collect()
    _check(_native.lib().fheon_release_memory())


def host_bootstrap_depth(config: ContextConfig) -> int:
    """Levels bootstrapping consumes under this configuration (CtS + EvalMod + StC)."""
    p = config.params()
    d = C.c_int()
    _check(_native.lib().fheon_host_bootstrap_depth(C.byref(p), C.byref(d)))
    return d.value


def host_security(config: ContextConfig) -> Dict[str, object]:
    """The security disclosure of a parameter set, computed on the host (no GPU)."""
    p = config.params()
    lq, lev, bound = C.c_double(), C.c_int(), C.c_double()
    _check(_native.lib().fheon_host_security(C.byref(p), C.byref(lq), C.byref(lev), C.byref(bound)))
    return security_report(config.ring_dimension, lq.value, lev.value, config)


def host_encode(config: ContextConfig, values, scale: float) -> np.ndarray:
    """Canonical-embedding encode on the host -> N signed integer coefficients."""
    p = config.params()
    v = np.ascontiguousarray(values, np.float64)
    out = np.zeros(config.ring_dimension, np.int64)
    _check(_native.lib().fheon_host_encode(C.byref(p), _dptr(v), v.size, float(scale),
                                           out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def cheb_relu_coefficients(beta: float, degree: int) -> np.ndarray:
    out = np.zeros(degree + 1, np.float64)
    _check(_native.lib().fheon_cheb_relu_coefficients(float(beta), int(degree), _dptr(out)))
    return out


def conv_depth_cost(cfg: ConvConfig, W_in: int) -> int:
    c = cfg.c()
    out = C.c_int()
    _check(_native.lib().fheon_conv_depth_cost(C.byref(c), W_in, C.byref(out)))
    return out.value
