"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the reference slotcnn core
compiled in place from /root/reference/proj (oracle/Makefile `make ref`,
output oracle/_ref/libslotcnn_ref.so, built by __graft_entry__.build() in the
container and shipped to the GPU box as a binary).

This is the decrypted-level oracle: the reference's own layer algorithms on
its cleartext slot simulator (proj/src/backend.cpp:165-249).  Import only
from tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libslotcnn_ref.so")
_lib = None

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_szp = C.POINTER(C.c_size_t)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle ref` where "
                               "/root/reference is present)")
        L = C.CDLL(LIB_PATH)
        L.sref_last_error.restype = C.c_char_p
        L.sref_backend_op.argtypes = [_sz, _sz, C.c_int, C.c_int, _dp, C.c_int, C.c_void_p, C.c_int, C.c_long, _dp,
                                      _ip, _lp, _sz, _szp]
        L.sref_convolution.argtypes = [_sz, _sz, C.c_int, _dp, C.c_int, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int,
                                       C.c_int, _dp, C.c_void_p, _dp, _ip, _szp, _szp, _lp, _sz, _szp]
        L.sref_pool.argtypes = [_sz, _sz, C.c_int, _dp, C.c_int, _sz, _sz, C.c_int, _sz, _sz, C.c_int, _dp, _ip,
                                _szp, _szp, _lp, _sz, _szp]
        L.sref_fully_connected.argtypes = [_sz, _sz, C.c_int, _dp, C.c_int, _sz, _sz, _sz, _dp, C.c_void_p, _dp,
                                           _ip, _lp, _sz, _szp]
        L.sref_secure_relu.argtypes = [_sz, _sz, C.c_int, _dp, C.c_int, C.c_double, C.c_int, _sz, _dp, _ip, _lp,
                                       _sz, _szp]
        L.sref_stride.argtypes = [_sz, _sz, C.c_int, _dp, C.c_int, _sz, _sz, _sz, C.c_int, _dp, _ip, _lp, _sz,
                                  _szp]
        L.sref_pad_input.argtypes = [_sz, _sz, C.c_int, _dp, C.c_int, _sz, _sz, _sz, _dp, _ip, _lp, _sz, _szp]
        L.sref_cheb_relu_coefficients.argtypes = [C.c_double, C.c_int, _dp]
        L.sref_cheb_eval_scalar.restype = C.c_double
        L.sref_cheb_eval_scalar.argtypes = [C.c_double, _dp, C.c_int]
        L.sref_depth_costs.argtypes = [_sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _sz, _ip]
        L.sref_time_convolution.argtypes = [_sz, _sz, C.c_int, _dp, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int,
                                            C.c_int, _dp, C.c_void_p, C.c_int, C.POINTER(C.c_double)]
        L.sref_time_rotate.argtypes = [_sz, _sz, C.c_int, C.c_long, C.c_int, C.POINTER(C.c_double)]
        L.sref_infer.argtypes = [C.c_char_p, _dp, _sz, _dp, _sz, _szp, C.POINTER(C.c_double), _ip, _sz, _szp,
                                 C.c_char_p, _sz, _lp, _sz, _szp]
        L.sref_layer_keys.argtypes = [C.c_char_p, _lp, _sz, _szp, _ip, _sz, _szp]
        L.sref_plan.argtypes = [C.c_int, _sz, _lp, _sz, _ip, _lp, _sz, _lp, _sz, _lp, _sz, _szp, _lp]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, msg, category):
        super().__init__(msg)
        self.category = category


_EV = {0: "rotation", 1: "mult_plain", 2: "mult_cipher", 3: "bootstrap"}
_EVCAP = 1 << 20


class Result:
    def __init__(self, slots, level, events, channels=None, width=None):
        self.slots = slots
        self.level = level
        self.events: List[Tuple[str, int]] = events
        self.channels = channels
        self.width = width

    def rotations(self):
        return [v for k, v in self.events if k == "rotation"]


class Ref:
    """The reference simulator with a given ring / slot count / depth budget."""

    def __init__(self, ring: int, slots: int, depth: int):
        self.ring, self.S, self.depth = ring, slots, depth

    def _ev(self):
        buf = np.zeros(2 * _EVCAP, dtype=np.int64)
        return buf, C.c_size_t()

    def _check(self, rc):
        if rc != 0:
            raise RefError(lib().sref_last_error().decode(), rc)

    @staticmethod
    def _events(buf, n):
        k = min(n.value, _EVCAP)
        return [(_EV[int(buf[2 * i])], int(buf[2 * i + 1])) for i in range(k)]

    def _full(self, x):
        v = np.zeros(self.S)
        x = np.asarray(x, np.float64).reshape(-1)
        v[: x.size] = x
        return v

    def convolution(self, x, level, C_, W, F, k, stride=1, pad=0, mode=0, variant=0, weights=None, bias=None):
        out = np.zeros(self.S)
        lvl = C.c_int()
        oc, ow = C.c_size_t(), C.c_size_t()
        buf, n = self._ev()
        w = np.ascontiguousarray(weights, np.float64).reshape(-1)
        b = None if bias is None else np.ascontiguousarray(bias, np.float64)
        self._check(lib().sref_convolution(self.ring, self.S, self.depth, self._full(x), level, C_, W, F, k, stride,
                                           pad, mode, variant, w, b.ctypes.data if b is not None else None, out,
                                           C.byref(lvl), C.byref(oc), C.byref(ow),
                                           buf.ctypes.data_as(_lp), _EVCAP, C.byref(n)))
        return Result(out, lvl.value, self._events(buf, n), oc.value, ow.value)

    def pool(self, x, level, C_, W, kind, k=2, stride=2, variant=0):
        out = np.zeros(self.S)
        lvl = C.c_int()
        oc, ow = C.c_size_t(), C.c_size_t()
        buf, n = self._ev()
        self._check(lib().sref_pool(self.ring, self.S, self.depth, self._full(x), level, C_, W, kind, k, stride,
                                    variant, out, C.byref(lvl), C.byref(oc), C.byref(ow), buf.ctypes.data_as(_lp),
                                    _EVCAP, C.byref(n)))
        return Result(out, lvl.value, self._events(buf, n), oc.value, ow.value)

    def fully_connected(self, x, level, n_in, m, merge_budget, weights, bias=None):
        out = np.zeros(self.S)
        lvl = C.c_int()
        buf, n = self._ev()
        w = np.ascontiguousarray(weights, np.float64).reshape(-1)
        b = None if bias is None else np.ascontiguousarray(bias, np.float64)
        self._check(lib().sref_fully_connected(self.ring, self.S, self.depth, self._full(x), level, n_in, m,
                                               merge_budget, w, b.ctypes.data if b is not None else None, out,
                                               C.byref(lvl), buf.ctypes.data_as(_lp), _EVCAP, C.byref(n)))
        return Result(out, lvl.value, self._events(buf, n))

    def secure_relu(self, x, level, scale=1.0, degree=59, active=0):
        out = np.zeros(self.S)
        lvl = C.c_int()
        buf, n = self._ev()
        self._check(lib().sref_secure_relu(self.ring, self.S, self.depth, self._full(x), level, scale, degree, active,
                                           out, C.byref(lvl), buf.ctypes.data_as(_lp), _EVCAP, C.byref(n)))
        return Result(out, lvl.value, self._events(buf, n))

    def stride(self, x, level, W, S_, W_out=0, variant=0):
        out = np.zeros(self.S)
        lvl = C.c_int()
        buf, n = self._ev()
        self._check(lib().sref_stride(self.ring, self.S, self.depth, self._full(x), level, W, S_, W_out, variant, out,
                                      C.byref(lvl), buf.ctypes.data_as(_lp), _EVCAP, C.byref(n)))
        return Result(out, lvl.value, self._events(buf, n))

    def pad_input(self, x, level, C_, W, P):
        out = np.zeros(self.S)
        lvl = C.c_int()
        buf, n = self._ev()
        self._check(lib().sref_pad_input(self.ring, self.S, self.depth, self._full(x), level, C_, W, P, out,
                                         C.byref(lvl), buf.ctypes.data_as(_lp), _EVCAP, C.byref(n)))
        return Result(out, lvl.value, self._events(buf, n))

    def backend_op(self, op, a, level_a, b=None, level_b=0, t=0):
        out = np.zeros(self.S)
        lvl = C.c_int()
        buf, n = self._ev()
        bb = self._full(b) if b is not None else None
        self._check(lib().sref_backend_op(self.ring, self.S, self.depth, op, self._full(a), level_a,
                                          bb.ctypes.data if bb is not None else None, level_b, t, out, C.byref(lvl),
                                          buf.ctypes.data_as(_lp), _EVCAP, C.byref(n)))
        return Result(out, lvl.value, self._events(buf, n))

    def time_convolution(self, x, C_, W, F, k, stride, pad, mode, variant, weights, bias, iters):
        sec = C.c_double()
        w = np.ascontiguousarray(weights, np.float64).reshape(-1)
        b = None if bias is None else np.ascontiguousarray(bias, np.float64)
        self._check(lib().sref_time_convolution(self.ring, self.S, self.depth,
                                                np.ascontiguousarray(x, np.float64).reshape(-1), C_, W, F, k, stride,
                                                pad, mode, variant, w, b.ctypes.data if b is not None else None,
                                                iters, C.byref(sec)))
        return sec.value

    def time_rotate(self, t, iters):
        sec = C.c_double()
        self._check(lib().sref_time_rotate(self.ring, self.S, self.depth, t, iters, C.byref(sec)))
        return sec.value


def infer(spec_path: str, x: np.ndarray, max_logits: int = 1 << 16):
    """The reference's build_model + infer (model_spec.cpp:864, model_run.cpp:100) on a
    spec JSON with CSV weights beside it.  Returns (logits, ledger rows
    [(name, level_in, level_out, is_bootstrap)], events, wall_ms)."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1)
    logits = np.zeros(max_logits)
    n = C.c_size_t()
    wall = C.c_double()
    ledger = np.zeros(3 * 4096, dtype=np.int32)
    nl = C.c_size_t()
    names = C.create_string_buffer(1 << 16)
    ev = np.zeros(2 * _EVCAP, dtype=np.int64)
    nev = C.c_size_t()
    rc = lib().sref_infer(spec_path.encode(), x, x.size, logits, max_logits, C.byref(n), C.byref(wall),
                          ledger.ctypes.data_as(_ip), 4096, C.byref(nl), names, len(names),
                          ev.ctypes.data_as(_lp), _EVCAP, C.byref(nev))
    if rc:
        raise RefError(lib().sref_last_error().decode(), rc)
    nm = names.value.decode().split("\n")
    rows = [(nm[i], int(ledger[3 * i]), int(ledger[3 * i + 1]), bool(ledger[3 * i + 2])) for i in range(nl.value)]
    events = Ref._events(ev, nev)
    return logits[: n.value].copy(), rows, events, wall.value


def cheb_relu_coefficients(beta: float, degree: int) -> np.ndarray:
    out = np.zeros(degree + 1)
    rc = lib().sref_cheb_relu_coefficients(beta, degree, out)
    if rc:
        raise RefError(lib().sref_last_error().decode(), rc)
    return out


def cheb_eval_scalar(x: float, coeffs: np.ndarray) -> float:
    c = np.ascontiguousarray(coeffs, np.float64)
    return lib().sref_cheb_eval_scalar(x, c, c.size)


def conv_depth_cost(C_, F, k, stride, pad, mode, variant, W_in) -> int:
    out = C.c_int()
    rc = lib().sref_depth_costs(C_, F, k, stride, pad, mode, variant, W_in, C.byref(out))
    if rc:
        raise RefError(lib().sref_last_error().decode(), rc)
    return out.value


def layer_keys(spec_path: str):
    """The reference's BuiltModel::layer_keys (model_spec.cpp:944-950) for a spec:
    [(usage dict {index: count}, ends_block)] per top-level layer."""
    cap = 1 << 16
    ent = np.zeros(3 * cap, dtype=np.int64)
    ends = np.zeros(4096, dtype=np.int32)
    ne, nl = C.c_size_t(), C.c_size_t()
    rc = lib().sref_layer_keys(spec_path.encode(), ent.ctypes.data_as(_lp), cap, C.byref(ne),
                               ends.ctypes.data_as(_ip), 4096, C.byref(nl))
    if rc:
        raise RefError(lib().sref_last_error().decode(), rc)
    out = [({}, bool(ends[i])) for i in range(nl.value)]
    for m in range(ne.value):
        out[int(ent[3 * m])][0][int(ent[3 * m + 1])] = int(ent[3 * m + 2])
    return out


def plan(mode: int, layers, ranges=(), events=()):
    """The reference's plan_single_block (0) / plan_blocks (1) / plan_blocks(ranges) (2)
    + verify_trace on `layers` [(usage dict, ends_block)] and `events` [(kind, value)]
    (kind 0 rotation, 4 "layer:<value>" marker).  Returns (blocks [(first, last, nkeys)],
    union size, peak resident, violations, unused keys, rotations checked)."""
    ent = [(i, k, c) for i, (u, _) in enumerate(layers) for k, c in sorted(u.items())]
    ent_a = np.array(ent if ent else [(0, 0, 0)], dtype=np.int64).reshape(-1)
    ends = np.array([int(e) for _, e in layers] or [0], dtype=np.int32)
    rg = np.array(list(ranges) or [(0, 0)], dtype=np.int64).reshape(-1)
    ev = np.array(list(events) or [(1, 0)], dtype=np.int64).reshape(-1)
    blocks = np.zeros(3 * 4096, dtype=np.int64)
    nb = C.c_size_t()
    out = np.zeros(5, dtype=np.int64)
    rc = lib().sref_plan(mode, len(layers), ent_a.ctypes.data_as(_lp), len(ent), ends.ctypes.data_as(_ip),
                         rg.ctypes.data_as(_lp), len(ranges), ev.ctypes.data_as(_lp), len(events),
                         blocks.ctypes.data_as(_lp), 4096, C.byref(nb), out.ctypes.data_as(_lp))
    if rc:
        raise RefError(lib().sref_last_error().decode(), rc)
    bl = [tuple(int(v) for v in blocks[3 * b:3 * b + 3]) for b in range(nb.value)]
    return bl, int(out[0]), int(out[1]), int(out[2]), int(out[3]), int(out[4])
