"""ctypes binding of the C ABI (include/fheon_b200.h).

The shared library is built in-tree (paper_2510_03996_b200/_lib/libfheon_b200.so,
see csrc/Makefile or __graft_entry__.build()).  There is no CPU fallback: if
the library is missing, or no CUDA device is visible, every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FHEON_LIB_OVERRIDE: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("FHEON_LIB_OVERRIDE") or os.path.join(_HERE, "_lib", "libfheon_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "fheon_b200.h")

_lib = None


class fheon_params(C.Structure):
    _fields_ = [
        ("log_n", C.c_int),
        ("limbs", C.c_int),
        ("special_limbs", C.c_int),
        ("dnum", C.c_int),
        ("first_mod_bits", C.c_int),
        ("scale_bits", C.c_int),
        ("special_bits", C.c_int),
        ("depth_budget", C.c_int),
        ("seed", C.c_uint64),
        ("hamming_weight", C.c_int),
        ("bootstrap", C.c_int),
        ("boot_scale_bits", C.c_int),
        ("digit_split", C.c_int),
        ("boot_hamming_weight", C.c_int),
        ("min_security", C.c_int),
        ("allow_insecure", C.c_int),
        ("no_secret", C.c_int),
        ("boot_k_range", C.c_int),
        ("boot_cts_levels", C.c_int),
        ("boot_stc_levels", C.c_int),
        ("boot_sparse", C.c_int),
    ]


class fheon_conv_cfg(C.Structure):
    _fields_ = [
        ("in_channels", C.c_size_t),
        ("out_channels", C.c_size_t),
        ("kernel", C.c_size_t),
        ("stride", C.c_size_t),
        ("padding", C.c_size_t),
        ("mode", C.c_int),
        ("stride_variant", C.c_int),
    ]


vp = C.c_void_p
pp = C.POINTER(C.c_void_p)
dp = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
szp = C.POINTER(C.c_size_t)
lp = C.POINTER(C.c_long)

# name -> (restype, argtypes)
SIGNATURES = {
    "fheon_last_error": (C.c_char_p, []),
    "fheon_last_error_kind": (C.c_int, []),
    "fheon_version": (C.c_int, []),
    "fheon_host_primes": (C.c_int, [C.POINTER(fheon_params), u64p, dp]),
    "fheon_host_security": (C.c_int, [C.POINTER(fheon_params), dp, C.POINTER(C.c_int), dp]),
    "fheon_host_bootstrap_depth": (C.c_int, [C.POINTER(fheon_params), C.POINTER(C.c_int)]),
    "fheon_ctx_security": (C.c_int, [vp, dp, C.POINTER(C.c_int)]),
    "fheon_ctx_clone": (C.c_int, [vp, C.POINTER(C.c_void_p)]),
    "fheon_release_memory": (C.c_int, []),
    "fheon_key_packed_words": (C.c_size_t, [vp]),
    "fheon_key_download_packed": (C.c_int, [vp, C.c_uint64, u64p]),
    "fheon_key_upload": (C.c_int, [vp, C.c_uint64, u64p]),
    "fheon_key_upload_packed": (C.c_int, [vp, C.c_uint64, u64p]),
    "fheon_key_upload_packed_async": (C.c_int, [vp, C.c_uint64, u64p]),
    "fheon_required_key_ids": (C.c_int, [vp, u64p, C.c_size_t, szp]),
    "fheon_key_uploads": (C.c_int, [vp, u64p, u64p]),
    "fheon_host_encode": (C.c_int, [C.POINTER(fheon_params), dp, C.c_size_t, C.c_double, C.POINTER(C.c_int64)]),
    "fheon_cheb_relu_coefficients": (C.c_int, [C.c_double, C.c_int, dp]),
    "fheon_ctx_create": (C.c_int, [C.POINTER(fheon_params), pp]),
    "fheon_ctx_destroy": (None, [vp]),
    "fheon_ctx_info": (C.c_int, [vp, u64p, dp, C.POINTER(C.c_int)]),
    "fheon_ctx_stream": (vp, [vp]),
    "fheon_ctx_sync": (C.c_int, [vp]),
    "fheon_ctx_stats": (C.c_int, [vp, u64p]),
    "fheon_ctx_reset_stats": (C.c_int, [vp]),
    "fheon_timer_arm": (C.c_int, [vp, C.c_int]),
    "fheon_timer_read": (C.c_int, [vp, dp, C.POINTER(C.c_int)]),
    "fheon_set_tracing": (C.c_int, [vp, C.c_int]),
    "fheon_trace": (C.c_int, [vp, lp, C.c_size_t, szp]),
    "fheon_trace_clear": (C.c_int, [vp]),
    "fheon_galois_elt": (C.c_uint64, [vp, C.c_long]),
    "fheon_keygen_rotations": (C.c_int, [vp, lp, C.c_size_t]),
    "fheon_keygen_relin": (C.c_int, [vp]),
    "fheon_set_strict_keys": (C.c_int, [vp, C.c_int]),
    "fheon_key_download": (C.c_int, [vp, C.c_uint64, u64p]),
    "fheon_key_count": (C.c_size_t, [vp]),
    "fheon_ct_free": (None, [vp]),
    "fheon_ct_level": (C.c_int, [vp]),
    "fheon_ct_limbs": (C.c_int, [vp]),
    "fheon_ct_scale": (C.c_double, [vp]),
    "fheon_encrypt": (C.c_int, [vp, dp, C.c_size_t, pp]),
    "fheon_encrypt_top": (C.c_int, [vp, dp, C.c_size_t, pp]),
    "fheon_decrypt": (C.c_int, [vp, vp, dp, C.c_size_t]),
    "fheon_decrypt_complex": (C.c_int, [vp, vp, dp, dp, C.c_size_t]),
    "fheon_ctx_depth_budget": (C.c_int, [vp]),
    "fheon_ctx_set_schedule": (C.c_int, [vp, C.c_int]),
    "fheon_ctx_schedule": (C.c_int, [vp]),
    "fheon_ctx_set_weight_cache": (C.c_int, [vp, C.c_uint64]),
    "fheon_ct_upload": (C.c_int, [vp, u64p, C.c_int, C.c_double, pp]),
    "fheon_ct_download": (C.c_int, [vp, vp, u64p]),
    "fheon_rotate": (C.c_int, [vp, vp, C.c_long, pp]),
    "fheon_rotate_hoisted": (C.c_int, [vp, vp, lp, C.c_size_t, pp]),
    "fheon_rotate_many": (C.c_int, [vp, pp, lp, C.c_size_t, pp]),
    "fheon_rotate_sum": (C.c_int, [vp, pp, lp, C.c_size_t, pp]),
    "fheon_ct_upload_async": (C.c_int, [vp, u64p, C.c_int, C.c_double, pp]),
    "fheon_ct_download_async": (C.c_int, [vp, vp, u64p]),
    "fheon_ct_packed_words": (C.c_size_t, [vp, C.c_int]),
    "fheon_key_bytes": (C.c_uint64, [vp]),
    "fheon_rotate_sum_many": (C.c_int, [vp, C.c_void_p, C.POINTER(C.c_long), C.POINTER(C.c_size_t), C.c_size_t,
                                        C.c_void_p]),
    "fheon_prefetch_rotation_keys": (C.c_int, [vp, C.POINTER(C.c_long), C.c_size_t]),
    "fheon_drop_rotation_keys": (C.c_int, [vp, C.POINTER(C.c_long), C.c_size_t]),
    "fheon_key_events": (C.c_int, [vp, u64p, u64p]),
    "fheon_ct_upload_packed": (C.c_int, [vp, u64p, C.c_int, C.c_double, pp]),
    "fheon_ct_download_packed": (C.c_int, [vp, vp, u64p]),
    "fheon_ct_upload_packed_async": (C.c_int, [vp, u64p, C.c_int, C.c_double, pp]),
    "fheon_ct_download_packed_async": (C.c_int, [vp, vp, u64p]),
    "fheon_ctx_wait_transfers": (C.c_int, [vp]),
    "fheon_add": (C.c_int, [vp, vp, vp, pp]),
    "fheon_sub": (C.c_int, [vp, vp, vp, pp]),
    "fheon_add_plain": (C.c_int, [vp, vp, dp, C.c_size_t, pp]),
    "fheon_mult_plain": (C.c_int, [vp, vp, dp, C.c_size_t, pp]),
    "fheon_mult_cipher": (C.c_int, [vp, vp, vp, pp]),
    "fheon_bootstrap": (C.c_int, [vp, vp, pp]),
    "fheon_bootstrap_active": (C.c_int, [vp, vp, C.c_size_t, C.c_int, pp]),
    "fheon_bootstrap_active_many": (C.c_int, [vp, pp, C.c_size_t, C.c_size_t, C.c_int, pp]),
    "fheon_bootstrap_stage": (C.c_int, [vp, vp, C.c_int, pp]),
    "fheon_bootstrap_info": (C.c_int, [vp, C.POINTER(C.c_int), dp, C.c_size_t, szp]),
    "fheon_rescale": (C.c_int, [vp, vp, pp]),
    "fheon_level_down": (C.c_int, [vp, vp, C.c_int, pp]),
    "fheon_keyswitch_raw": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, pp]),
    "fheon_ntt_host": (C.c_int, [vp, u64p, C.c_int, C.c_int, C.c_int]),
    "fheon_automorph_host": (C.c_int, [vp, u64p, C.c_int, C.c_int, C.c_uint64]),
    "fheon_microbench": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp]),
    "fheon_convolution": (C.c_int, [vp, vp, C.c_size_t, C.c_size_t, C.POINTER(fheon_conv_cfg), dp, dp, pp, szp,
                                    szp]),
    "fheon_pool": (C.c_int, [vp, vp, C.c_size_t, C.c_size_t, C.c_int, C.c_size_t, C.c_size_t, C.c_int, pp, szp,
                             szp]),
    "fheon_fully_connected": (C.c_int, [vp, vp, C.c_size_t, C.c_size_t, C.c_size_t, dp, dp, pp]),
    "fheon_secure_relu": (C.c_int, [vp, vp, C.c_double, C.c_int, C.c_size_t, pp]),
    "fheon_secure_relu_many": (C.c_int, [vp, pp, C.c_size_t, C.c_double, C.c_int, C.c_size_t, pp]),
    "fheon_stride": (C.c_int, [vp, vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, pp]),
    "fheon_pad_input": (C.c_int, [vp, vp, C.c_size_t, C.c_size_t, C.c_size_t, pp]),
    "fheon_conv_depth_cost": (C.c_int, [C.POINTER(fheon_conv_cfg), C.c_size_t, C.POINTER(C.c_int)]),
}


def lib():
    """Load the in-tree shared library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"B200 engine library not built: {LIB_PATH} (run `make -C paper_2510_03996_b200/csrc` "
                "or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def header_symbols():
    """Function names declared in include/fheon_b200.h."""
    import re
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(fheon_[a-z0-9_]+)\s*\(", text)))
