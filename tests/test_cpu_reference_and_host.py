"""CPU tests: the reference oracle, golden fixtures, host-side engine logic
(prime chain, encoder, Chebyshev coefficients, depth costs) and the C ABI
surface -- no device compute is invoked.
"""
import json
import os

import numpy as np
import pytest

import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import _native
from oracle import ref as sref
from oracle.ckks_oracle import Oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
need_ref = pytest.mark.skipif(not sref.available(), reason="oracle/_ref not built")


def _ev(events):
    kinds = {"rotation": 0, "mult_plain": 1, "mult_cipher": 2, "bootstrap": 3}
    return np.array([(kinds[k], v) for k, v in events], dtype=np.int64).reshape(-1, 2)


# ------------------------------------------------------------ C ABI surface
def test_library_exports_every_header_symbol():
    lib = _native.lib()
    syms = _native.header_symbols()
    assert len(syms) >= 50
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/fheon_b200.h but not exported"
    assert set(syms) <= set(_native.SIGNATURES), "ctypes signatures missing for some header symbols"


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except ImportError:
        pass
    with pytest.raises(fh.CudaError, match="no CUDA device"):
        fh.SlotContext(fh.ContextConfig.preset("config1"))


# ------------------------------------------------------------ host logic
@pytest.mark.parametrize("preset,logn", [("config1", 14), ("config2", 16)])
def test_host_prime_chain_matches_oracle(preset, logn):
    cfg = fh.ContextConfig.preset(preset)
    primes, scales = fh.api.host_primes(cfg)
    c = cfg.crypto
    o = Oracle(logn, cfg.limbs, cfg.special_limbs, c.key_switch_digits, c.first_modulus_bits, c.rescale_bits,
               cfg.special_bits, 1)
    assert np.array_equal(primes, o.primes)
    assert np.array_equal(scales, o.T)


def test_host_encoder_matches_oracle_bit_exact():
    cfg = fh.ContextConfig(4096, 2048, 5, fh.CryptoMetadata(50, 40, 3), limbs=6, special_limbs=2)
    o = Oracle(12, 6, 2, 3, 50, 40, 60, 1)
    rng = np.random.default_rng(0)
    for n in (2048, 100, 1):
        v = rng.uniform(-3, 3, n)
        assert np.array_equal(fh.api.host_encode(cfg, v, 2.0 ** 40), o.encode_coeffs(v, 2.0 ** 40))


def test_parameter_validation():
    bad = fh.ContextConfig(4096, 2048, 13, fh.CryptoMetadata(50, 40, 3), limbs=14, special_limbs=1)
    with pytest.raises(fh.ShapeError):
        fh.api.host_primes(fh.ContextConfig(4096, 1000, 5))
    # engine-side checks (P must dominate every digit) happen at context creation; host tables still build
    fh.api.host_primes(bad)


@need_ref
@pytest.mark.parametrize("beta,degree", [(1.0, 59), (8.0, 59), (1.0, 7), (3.5, 27)])
def test_cheb_coefficients_bit_exact_vs_reference(beta, degree):
    assert np.array_equal(fh.api.cheb_relu_coefficients(beta, degree), sref.cheb_relu_coefficients(beta, degree))


def test_relu_epsilon59_frozen_bound():
    """Reference fixture proj/tests/data/relu_epsilon59.json (acceptance criterion 5)."""
    fx = json.load(open(os.path.join(GOLDEN, "relu_epsilon59.json")))
    c = fh.api.cheb_relu_coefficients(1.0, fx["degree"])
    z = np.linspace(-1, 1, fx["grid_points"])
    # Clenshaw evaluation of the series
    b1 = np.zeros_like(z)
    b2 = np.zeros_like(z)
    for d in range(len(c) - 1, 0, -1):
        b1, b2 = c[d] + 2 * z * b1 - b2, b1
    p = c[0] + z * b1 - b2
    err = np.abs(p - np.maximum(z, 0))
    assert err.max() <= fx["sup_norm"]
    assert err[np.abs(z) >= fx["deadzone"]].max() <= fx["epsilon_59"]


@pytest.mark.parametrize("C,F,k,S,P,mode,variant,W", [(1, 6, 5, 1, 0, 0, 0, 28), (3, 4, 3, 1, 1, 1, 0, 8),
                                                       (2, 4, 2, 2, 0, 0, 1, 8), (2, 4, 3, 1, 1, 0, 0, 6),
                                                       (2, 4, 2, 2, 0, 2, 0, 8)])
def test_conv_depth_cost_matches_reference(C, F, k, S, P, mode, variant, W):
    got = fh.conv_depth_cost(fh.ConvConfig(C, F, k, S, P, fh.ConvMode(mode), fh.StrideVariant(variant)), W)
    if sref.available():
        assert got == sref.conv_depth_cost(C, F, k, S, P, mode, variant, W)
    assert got >= 2


# ------------------------------------------------------------ reference oracle + golden
@need_ref
def test_reference_reproduces_golden_config1():
    g = np.load(os.path.join(GOLDEN, "conv_config1.npz"))
    r = sref.Ref(16384, 8192, 10).convolution(g["x"], 10, 1, 28, 6, 5, 1, 0, 0, 0, g["w"], None)
    assert np.array_equal(r.slots[: 6 * 24 * 24], g["out"])
    assert r.level == int(g["level"]) == 7
    assert np.array_equal(_ev(r.events), g["events"])
    rots = [v for k, v in r.events if k == "rotation"]
    assert len(rots) == 305 and len(set(rots)) == 52


@need_ref
def test_reference_golden_small_layers():
    r = sref.Ref(4096, 2048, 13)
    g = np.load(os.path.join(GOLDEN, "special3x3_small.npz"))
    res = r.convolution(g["x"], 13, 3, 8, 4, 3, 1, 1, 1, 0, g["w"], g["b"])
    assert np.array_equal(res.slots, g["out"]) and np.array_equal(_ev(res.events), g["events"])
    g = np.load(os.path.join(GOLDEN, "relu59_beta8_small.npz"))
    res = r.secure_relu(g["x"], 13, 8.0, 59, 40)
    assert np.array_equal(res.slots, g["out"]) and res.level == int(g["level"])


@need_ref
def test_oracle_ops_agree_with_reference_simulator():
    """Decrypted-level parity of the CPU CKKS oracle with slotcnn's backend ops
    (rotation direction, mult_plain, mult_cipher, add; backend.cpp:165-231)."""
    o = Oracle(12, 6, 2, 3, 50, 40, 60, 3)
    r = sref.Ref(4096, 2048, 5)
    rng = np.random.default_rng(12)
    a, b = rng.uniform(-1, 1, o.S), rng.uniform(-1, 1, o.S)
    ca, cb = o.encrypt(a, 0), o.encrypt(b, 1)
    for t in (1, -3, 100):
        want = r.backend_op(0, a, 5, t=t)
        got = o.decrypt(o.rotate(ca, t, o.rotation_key(t)), o.T[-1])
        assert np.abs(got - want.slots).max() < 1e-6 and want.level == 5
    want = r.backend_op(3, a, 5, b=b)
    mp, s = o.mult_plain(ca, o.T[-1], b)
    assert np.abs(o.decrypt(mp, s) - want.slots).max() < 1e-6 and want.level == mp.shape[1] - 1
    want = r.backend_op(4, a, 5, b=b, level_b=5)
    mc = o.mult_cipher(ca, cb, o.relin_key())
    assert np.abs(o.decrypt(mc, o.T[-1] ** 2 / float(o.primes[5])) - want.slots).max() < 1e-6
    assert want.level == mc.shape[1] - 1
    want = r.backend_op(1, a, 5, b=b, level_b=3)
    cb3, s3 = o.level_down(cb, o.T[-1], 4)
    ca3, _ = o.level_down(ca, o.T[-1], 4)
    assert np.abs(o.decrypt(o.add(ca3, cb3), s3) - want.slots).max() < 1e-6 and want.level == 3


# ------------------------------------------------------------ model runtime (host logic)
def _flat_ledger(layers):
    from paper_2510_03996_b200 import model as M
    out = []
    for b in layers:
        out.append((b.name, b.type == "bootstrap"))
    return out


@pytest.mark.parametrize("budget,want", [(25, 3), (16, 4), (12, 5), (10, 6), (9, 8)])
def test_lenet_bootstrap_placement_counts(budget, want):
    """Standard placement + ledger repair (model_spec.cpp:746-851) give the
    reference's bootstrap counts."""
    from paper_2510_03996_b200 import model as M
    assert M.count_bootstraps(M.build(M.lenet5(ring=8192, depth_budget=budget))) == want


@pytest.mark.parametrize("budget,want", [(25, 18), (12, 19), (10, 22), (9, 38)])
def test_resnet_bootstrap_placement_counts(budget, want):
    from paper_2510_03996_b200 import model as M
    assert M.count_bootstraps(M.build(M.resnet20(ring=65536, depth_budget=budget))) == want


@need_ref
@pytest.mark.parametrize("budget", [25, 12, 9])
def test_lenet_ledger_matches_reference(budget, tmp_path):
    """Layer order (incl. inserted bootstraps) and per-layer declared costs match
    the reference's build; levels are checked on the GPU."""
    from paper_2510_03996_b200 import model as M
    spec = M.lenet5(ring=8192, depth_budget=budget)
    path = spec.write(str(tmp_path))
    x = np.random.default_rng(1).uniform(0, 1, (1, 28, 28))
    _, rows, _, _ = sref.infer(path, x)
    layers = M.build(spec)
    assert [b.name for b in layers] == [r[0] for r in rows]
    level = budget
    for b, r in zip(layers, rows):
        assert r[1] == level
        level = budget if b.type == "bootstrap" else level - b.cost
        assert r[2] == level


def test_security_disclosure_and_secure_chains():
    """HE-standard security (homomorphicencryption.org 2018, uniform ternary):
    configs[1] (log2 QP 1690 at N = 2^16) meets 128 bits; configs[0] (690 > 438
    at N = 2^14) and the reference's presets do not (they carry allow_insecure);
    the model runtime's default ResNet-20 chain at depth 12 meets 128 bits with a
    dense secret, and refuses depth 25 (log2 Q alone exceeds the bound)."""
    from paper_2510_03996_b200 import model as M
    s2 = fh.host_security(fh.ContextConfig.preset("config2"))
    assert s2["meets_128"] and s2["security_bits"] == 128 and abs(s2["log2_qp"] - 1690) < 5
    s1 = fh.host_security(fh.ContextConfig.preset("config1"))
    assert not s1["meets_128"] and s1["security_bits"] == 0
    assert fh.ContextConfig.preset("config1").allow_insecure and fh.ContextConfig.preset("large").allow_insecure
    cfg = M.ckks_config(M.resnet20(ring=65536, depth_budget=12), True)
    sec = fh.host_security(cfg)
    assert cfg.hamming_weight == 0 and sec["meets_128"] and sec["log2_qp"] <= 1747
    assert "encapsulation" in sec["secret"]
    with pytest.raises(fh.ModelError, match="no 128-bit chain"):
        M.ckks_config(M.resnet20(ring=65536, depth_budget=25), True)
    ins = M.ckks_config(M.resnet20(ring=65536, depth_budget=25), True, security=0)
    si = fh.host_security(ins)
    assert si["security_bits"] is None and not si["meets_128"] and si["log2_qp"] > 2600  # sparse h=64 main secret


def test_integration_seam_links_the_engine_not_the_simulator():
    """integration/_build/libslotcnn_b200.so: the reference core compiled against
    integration/include/slotcnn/backend.hpp -- its backend entry points are
    defined by backend_b200.cpp and call the C ABI (fheon_*), and the reference
    simulator's backend.cpp is not in it."""
    import subprocess
    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                       "libslotcnn_b200.so")
    if not os.path.exists(lib):
        pytest.skip("integration not built (needs /root/reference: make -C integration)")
    syms = subprocess.run(["nm", "-DC", lib], capture_output=True, text=True).stdout
    defined = {ln.split(" ", 2)[-1] for ln in syms.splitlines() if " T " in ln}
    undefined = {ln.split()[-1] for ln in syms.splitlines() if " U " in ln}
    for fn in ("slotcnn::rotate(slotcnn::SlotVector const&, long)", "slotcnn::bootstrap(slotcnn::SlotVector const&)",
               "slotcnn::convolution(slotcnn::PackedTensor const&, slotcnn::ConvConfig const&, "
               "slotcnn::KernelTensor const&)"):
        assert fn in defined, fn
    for fn in ("fheon_rotate", "fheon_mult_cipher", "fheon_bootstrap", "fheon_ctx_create"):
        assert fn in undefined, fn
    assert "slotcnn::SlotVector::slots() const" in defined  # decrypt-on-read (backend_b200.cpp)


def test_he_standard_table_and_chain_properties():
    """The HE-standard bounds the engine enforces (homomorphicencryption.org 2018 Table 1,
    ternary, classical; 2^16 as OpenFHE ships it), and the 128-bit chains the model
    runtime builds: dense secret, encapsulation h_b = 32 with EvalMod range 12 (a
    15-level bootstrap), log2 QP under the bound, the fewest digits that fit."""
    from paper_2510_03996_b200 import model as M
    for logn, bound in ((14, 438), (15, 881), (16, 1747)):
        cfg = fh.ContextConfig(1 << logn, 1 << (logn - 1), 5, fh.CryptoMetadata(50, 40, 3), limbs=6,
                               special_limbs=2, allow_insecure=True)
        assert fh.host_security(cfg)["he_standard_128_bound"] == bound
    prev_dnum = None
    for depth in (9, 10, 11, 12):
        cfg = M.ckks_config(M.resnet20(ring=65536, depth_budget=depth), True)
        sec = fh.host_security(cfg)
        assert sec["meets_128"] and sec["log2_qp"] <= 1747
        assert cfg.hamming_weight == 0 and cfg.boot_hamming_weight == 32 and cfg.boot_k_range == 12
        assert fh.host_bootstrap_depth(cfg) == 15 and cfg.limbs == depth + 1 + 15
        prev_dnum = cfg.crypto.key_switch_digits
    assert prev_dnum is not None


def test_oracle_encapsulation_keys_structure():
    """The oracle's restatement of the sparse-secret encapsulation keys: key 2 (s -> s_b)
    exists only on digit 0's q_0 limb and the special primes, and switching a level-0
    ciphertext with it and back (key 4 at level 0) preserves the decryption."""
    o = Oracle(12, 6, 2, 3, 50, 40, 60, 9)
    o.set_boot_secret(32)
    k2, k4 = o.keygen(2), o.keygen(4)
    assert not k2[1:].any() and not k2[0, :, 1:6].any() and k2[0, :, 0].any() and k2[0, :, 6:].any()
    assert k4[0, :, 0].any() and k4[2].any()
    rng = np.random.default_rng(2)
    v = rng.uniform(-1, 1, o.S)
    ct = o.encrypt(v, 0)
    c1 = np.ascontiguousarray(ct[:, :1])
    ks0, ks1 = o.keyswitch(np.ascontiguousarray(c1[1]), k2, 1)  # now under s_b
    y = np.stack([(c1[0].astype(object) + ks0.astype(object)) % int(o.primes[0]), ks1.astype(object)])
    y = np.ascontiguousarray(y.astype(np.uint64))
    back0, back1 = o.keyswitch(np.ascontiguousarray(y[1]), k4, 1)  # s_b -> s
    z = np.stack([(y[0].astype(object) + back0.astype(object)) % int(o.primes[0]), back1.astype(object)])
    z = np.ascontiguousarray(z.astype(np.uint64))
    assert np.abs(o.decrypt(z, float(o.T[0])) - o.decrypt(c1, float(o.T[0]))).max() < 1e-6


def test_bench_arms_print_the_same_config():
    """The two bench arms' `config` dicts are built by one function (same_config)."""
    import bench
    assert bench.head_config(11) == bench.head_config(11)
    assert bench.head_config(11)["workload"].startswith("configs[3]")
