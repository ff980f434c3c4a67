"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the CPU RNS-CKKS oracle
(oracle/ckks_oracle.c).  Import only from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  See ckks_oracle.h for the
parity status of the restatement.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libckks_oracle.so")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_dblp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"CKKS oracle not built: {_LIB_PATH} (run `make -C oracle ckks`)")
        L = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        L.ock_create.restype = vp
        L.ock_create.argtypes = [C.c_int] * 7 + [C.c_uint64]
        L.ock_create_chain.restype = vp
        L.ock_create_chain.argtypes = [C.c_int] * 4 + [_u64p, _dblp, C.c_uint64]
        L.ock_destroy.argtypes = [vp]
        L.ock_info.argtypes = [vp, _u64p, _u64p, _dblp]
        L.ock_ntt_fwd.argtypes = [vp, C.c_int, _u64p]
        L.ock_ntt_inv.argtypes = [vp, C.c_int, _u64p]
        L.ock_ntt_naive.argtypes = [vp, C.c_int, _u64p, _u64p]
        L.ock_negacyclic_mul_naive.argtypes = [vp, C.c_int, _u64p, _u64p, _u64p]
        L.ock_ntt_fwd_limbs.argtypes = [vp, _u64p, C.c_int, C.c_void_p]
        L.ock_ntt_inv_limbs.argtypes = [vp, _u64p, C.c_int, C.c_void_p]
        L.ock_automorph_ntt.argtypes = [vp, C.c_uint64, _u64p, _u64p, C.c_int]
        L.ock_automorph_coeff.argtypes = [vp, C.c_uint64, _u64p, _u64p, C.c_int, C.c_void_p]
        L.ock_galois_elt.restype = C.c_uint64
        L.ock_galois_elt.argtypes = [vp, C.c_long]
        L.ock_encode.argtypes = [vp, _dblp, C.c_size_t, C.c_int, C.c_double, _u64p]
        L.ock_encode_coeffs.argtypes = [vp, _dblp, C.c_size_t, C.c_double, _i64p]
        L.ock_decode_coeffs.argtypes = [vp, _dblp, C.c_double, _dblp]
        L.ock_secret.argtypes = [vp, _i8p]
        L.ock_set_hamming_weight.argtypes = [vp, C.c_int]
        L.ock_set_digit_split.argtypes = [vp, C.c_int]
        L.ock_set_boot_secret.argtypes = [vp, C.c_int]
        L.ock_keygen.argtypes = [vp, C.c_uint64, _u64p]
        L.ock_encrypt.argtypes = [vp, _dblp, C.c_size_t, C.c_uint64, _u64p]
        L.ock_decrypt.argtypes = [vp, _u64p, C.c_int, C.c_double, _dblp]
        L.ock_modup.argtypes = [vp, _u64p, C.c_int, _u64p]
        L.ock_moddown.argtypes = [vp, _u64p, C.c_int, _u64p]
        L.ock_keyswitch.argtypes = [vp, _u64p, C.c_int, _u64p, C.c_uint64, _u64p, _u64p]
        L.ock_rotate.argtypes = [vp, _u64p, C.c_int, C.c_long, _u64p, _u64p]
        L.ock_rotate_sum.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, _u64p]
        L.ock_rescale.argtypes = [vp, _u64p, C.c_int, _u64p]
        L.ock_rescale_poly.argtypes = [vp, _u64p, C.c_int, _u64p]
        L.ock_add.argtypes = [vp, _u64p, _u64p, C.c_int, C.c_int, _u64p]
        L.ock_sub.argtypes = [vp, _u64p, _u64p, C.c_int, C.c_int, _u64p]
        L.ock_mul_pt.argtypes = [vp, _u64p, _u64p, C.c_int, C.c_int, _u64p]
        L.ock_mult_plain.argtypes = [vp, _u64p, C.c_int, C.c_double, _dblp, C.c_size_t, _u64p,
                                     C.POINTER(C.c_double)]
        L.ock_mult_cipher.argtypes = [vp, _u64p, _u64p, C.c_int, _u64p, _u64p]
        L.ock_level_down.argtypes = [vp, _u64p, C.c_int, C.c_double, C.c_int, _u64p,
                                     C.POINTER(C.c_double)]
        L.ock_packed_words.argtypes = [vp, C.c_int]
        L.ock_packed_words.restype = C.c_size_t
        L.ock_pack.argtypes = [vp, _u64p, C.c_int, _u64p]
        L.ock_unpack.argtypes = [vp, _u64p, C.c_int, _u64p]
        _lib = L
    return _lib


def _chk(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with rc={rc}")


class Oracle:
    """CPU RNS-CKKS context mirroring the engine's parameter spec."""

    def __init__(self, logN, L, K, dnum, first_bits=0, scale_bits=0, special_bits=0, seed=1, hamming_weight=0,
                 digit_split=0, chain=None):
        self.logN, self.L, self.K, self.dnum = logN, L, K, dnum
        self.N = 1 << logN
        self.S = self.N // 2
        self.alpha = (L + dnum - 1) // dnum
        if chain is not None:
            primes, T = chain
            self._c = lib().ock_create_chain(logN, L, K, dnum, np.ascontiguousarray(primes, np.uint64),
                                             np.ascontiguousarray(T, np.float64), seed)
        else:
            self._c = lib().ock_create(logN, L, K, dnum, first_bits, scale_bits, special_bits, seed)
        if not self._c:
            raise ValueError("invalid oracle parameters")
        self.primes = np.zeros(L + K, np.uint64)
        self.psi = np.zeros(L + K, np.uint64)
        self.T = np.zeros(L, np.float64)
        lib().ock_info(self._c, self.primes, self.psi, self.T)
        if hamming_weight:
            lib().ock_set_hamming_weight(self._c, int(hamming_weight))
        if digit_split:
            _chk(lib().ock_set_digit_split(self._c, 1), "set_digit_split")

    @classmethod
    def from_chain(cls, logN, primes, T, L, K, dnum, seed=1, hamming_weight=0, digit_split=0):
        """Oracle over an explicit prime chain (e.g. the engine context's own:
        ctx.primes, ctx.scales) -- for the model runtime's mixed-width chains."""
        return cls(logN, L, K, dnum, seed=seed, hamming_weight=hamming_weight, digit_split=digit_split,
                   chain=(np.asarray(primes, np.uint64)[:L + K], np.asarray(T, np.float64)[:L]))

    def __del__(self):
        if getattr(self, "_c", None):
            lib().ock_destroy(self._c)
            self._c = None

    # ---- NTT
    def ntt(self, a, pi):
        a = np.ascontiguousarray(a, np.uint64).copy()
        lib().ock_ntt_fwd(self._c, pi, a)
        return a

    def intt(self, a, pi):
        a = np.ascontiguousarray(a, np.uint64).copy()
        lib().ock_ntt_inv(self._c, pi, a)
        return a

    def ntt_limbs(self, a, inverse=False, limb_map=None):
        a = np.ascontiguousarray(a, np.uint64).copy()
        n = a.size // self.N
        m = None
        if limb_map is not None:
            mm = (C.c_int * n)(*limb_map)
            m = C.cast(mm, C.c_void_p)
        (lib().ock_ntt_inv_limbs if inverse else lib().ock_ntt_fwd_limbs)(self._c, a.reshape(-1), n, m)
        return a

    def ntt_naive(self, a, pi):
        out = np.zeros(self.N, np.uint64)
        lib().ock_ntt_naive(self._c, pi, np.ascontiguousarray(a, np.uint64), out)
        return out

    def negacyclic_mul_naive(self, a, b, pi):
        out = np.zeros(self.N, np.uint64)
        lib().ock_negacyclic_mul_naive(self._c, pi, np.ascontiguousarray(a, np.uint64),
                                       np.ascontiguousarray(b, np.uint64), out)
        return out

    # ---- automorphism
    def galois(self, t):
        return int(lib().ock_galois_elt(self._c, int(t)))

    def automorph_ntt(self, a, g):
        a = np.ascontiguousarray(a, np.uint64)
        out = np.zeros_like(a)
        lib().ock_automorph_ntt(self._c, g, a.reshape(-1), out.reshape(-1), a.size // self.N)
        return out

    def automorph_coeff(self, a, g):
        a = np.ascontiguousarray(a, np.uint64)
        out = np.zeros_like(a)
        lib().ock_automorph_coeff(self._c, g, a.reshape(-1), out.reshape(-1), a.size // self.N, None)
        return out

    # ---- encoder
    def encode(self, vals, limbs, scale):
        v = np.ascontiguousarray(vals, np.float64)
        out = np.zeros((limbs, self.N), np.uint64)
        _chk(lib().ock_encode(self._c, v, v.size, limbs, scale, out), "encode")
        return out

    def encode_coeffs(self, vals, scale):
        v = np.ascontiguousarray(vals, np.float64)
        out = np.zeros(self.N, np.int64)
        _chk(lib().ock_encode_coeffs(self._c, v, v.size, scale, out), "encode_coeffs")
        return out

    def decode_coeffs(self, coeffs, scale):
        out = np.zeros(self.S, np.float64)
        lib().ock_decode_coeffs(self._c, np.ascontiguousarray(coeffs, np.float64), scale, out)
        return out

    # ---- keys / encryption
    def secret(self):
        s = np.zeros(self.N, np.int8)
        lib().ock_secret(self._c, s)
        return s

    def set_boot_secret(self, hb=64):
        """sparse-secret encapsulation: key ids 2 (s -> s_b) and 4 (s_b -> s)"""
        lib().ock_set_boot_secret(self._c, int(hb))

    def keygen(self, key_id):
        key = np.zeros((self.dnum, 2, self.L + self.K, self.N), np.uint64)
        _chk(lib().ock_keygen(self._c, key_id, key), "keygen")
        return key

    def rotation_key(self, t):
        return self.keygen(self.galois(t))

    def relin_key(self):
        return self.keygen(0)

    def encrypt(self, vals, counter=0):
        v = np.ascontiguousarray(vals, np.float64)
        ct = np.zeros((2, self.L, self.N), np.uint64)
        _chk(lib().ock_encrypt(self._c, v, v.size, counter, ct), "encrypt")
        return ct

    def decrypt(self, ct, scale):
        ct = np.ascontiguousarray(ct, np.uint64)
        limbs = ct.shape[1]
        out = np.zeros(self.S, np.float64)
        _chk(lib().ock_decrypt(self._c, ct, limbs, scale, out), "decrypt")
        return out

    # ---- key switching
    def modup(self, d):
        d = np.ascontiguousarray(d, np.uint64)
        limbs = d.shape[0]
        beta = (limbs + self.alpha - 1) // self.alpha
        out = np.zeros((beta, limbs + self.K, self.N), np.uint64)
        _chk(lib().ock_modup(self._c, d, limbs, out), "modup")
        return out

    def moddown(self, acc):
        acc = np.ascontiguousarray(acc, np.uint64)
        limbs = acc.shape[0] - self.K
        out = np.zeros((limbs, self.N), np.uint64)
        _chk(lib().ock_moddown(self._c, acc, limbs, out), "moddown")
        return out

    def keyswitch(self, d, key, g=1):
        d = np.ascontiguousarray(d, np.uint64)
        limbs = d.shape[0]
        ks0 = np.zeros((limbs, self.N), np.uint64)
        ks1 = np.zeros((limbs, self.N), np.uint64)
        _chk(lib().ock_keyswitch(self._c, d, limbs, np.ascontiguousarray(key), g, ks0, ks1), "keyswitch")
        return ks0, ks1

    # ---- evaluator
    def rotate(self, ct, t, key):
        ct = np.ascontiguousarray(ct, np.uint64)
        out = np.zeros_like(ct)
        _chk(lib().ock_rotate(self._c, ct, ct.shape[1], int(t), np.ascontiguousarray(key), out), "rotate")
        return out

    def rotate_sum(self, cts, ts, keys):
        """sum_j rotate(cts[j], ts[j]) with one ModDown (ckks_oracle.c ock_rotate_sum)."""
        cts = [np.ascontiguousarray(c, np.uint64) for c in cts]
        keys = [np.ascontiguousarray(k, np.uint64) for k in keys]
        n = len(cts)
        limbs = cts[0].shape[1]
        cp = (C.c_void_p * n)(*[c.ctypes.data for c in cts])
        kp = (C.c_void_p * n)(*[k.ctypes.data for k in keys])
        tp = (C.c_long * n)(*[int(t) for t in ts])
        out = np.zeros((2, limbs, self.N), np.uint64)
        _chk(lib().ock_rotate_sum(self._c, cp, tp, n, limbs, kp, out), "rotate_sum")
        return out

    def pack(self, ct):
        """packed wire format words of a [2][limbs][N] ciphertext"""
        ct = np.ascontiguousarray(ct, np.uint64)
        limbs = ct.shape[1]
        out = np.zeros(lib().ock_packed_words(self._c, limbs), np.uint64)
        lib().ock_pack(self._c, ct, limbs, out)
        return out

    def unpack(self, words, limbs):
        words = np.ascontiguousarray(words, np.uint64)
        out = np.zeros((2, limbs, self.N), np.uint64)
        lib().ock_unpack(self._c, words, limbs, out)
        return out

    def rescale(self, ct):
        ct = np.ascontiguousarray(ct, np.uint64)
        limbs = ct.shape[1]
        out = np.zeros((2, limbs - 1, self.N), np.uint64)
        _chk(lib().ock_rescale(self._c, ct, limbs, out), "rescale")
        return out

    def add(self, a, b):
        a = np.ascontiguousarray(a, np.uint64)
        out = np.zeros_like(a)
        lib().ock_add(self._c, a, np.ascontiguousarray(b, np.uint64), a.shape[0], a.shape[1], out)
        return out

    def sub(self, a, b):
        a = np.ascontiguousarray(a, np.uint64)
        out = np.zeros_like(a)
        lib().ock_sub(self._c, a, np.ascontiguousarray(b, np.uint64), a.shape[0], a.shape[1], out)
        return out

    def mul_pt(self, a, pt):
        a = np.ascontiguousarray(a, np.uint64)
        out = np.zeros_like(a)
        lib().ock_mul_pt(self._c, a, np.ascontiguousarray(pt, np.uint64), a.shape[0], a.shape[1], out)
        return out

    def mult_plain(self, ct, scale, vals):
        ct = np.ascontiguousarray(ct, np.uint64)
        limbs = ct.shape[1]
        v = np.ascontiguousarray(vals, np.float64)
        out = np.zeros((2, limbs - 1, self.N), np.uint64)
        s = C.c_double()
        _chk(lib().ock_mult_plain(self._c, ct, limbs, scale, v, v.size, out, C.byref(s)), "mult_plain")
        return out, s.value

    def mult_cipher(self, a, b, rk):
        a = np.ascontiguousarray(a, np.uint64)
        limbs = a.shape[1]
        out = np.zeros((2, limbs - 1, self.N), np.uint64)
        _chk(lib().ock_mult_cipher(self._c, a, np.ascontiguousarray(b, np.uint64), limbs,
                                   np.ascontiguousarray(rk), out), "mult_cipher")
        return out

    def level_down(self, ct, scale, target_limbs):
        ct = np.ascontiguousarray(ct, np.uint64)
        out = np.zeros((2, target_limbs, self.N), np.uint64)
        s = C.c_double()
        _chk(lib().ock_level_down(self._c, ct, ct.shape[1], scale, target_limbs, out, C.byref(s)),
             "level_down")
        return out, s.value
