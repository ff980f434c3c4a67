"""GPU: encrypted end-to-end inference through the model runtime against the
reference's own build_model() + infer() (oracle/_ref) on the same spec,
weights and input: same bootstrap placement, same per-layer ledger, same
event multiset, decrypted logits within max-abs 1e-3 (north-star tolerance).
"""
import tempfile

import numpy as np
import pytest

from paper_2510_03996_b200 import model as M
from oracle import ref as sref

pytestmark = pytest.mark.gpu


def _compare(spec, x, schedule="reference", security=0):
    """security=0: the insecure chains the reference's presets / toy rings need
    (disclosed); security=128: the HE-standard 128-bit chain (dense secret,
    sparse-secret encapsulation)."""
    path = spec.write(tempfile.mkdtemp())
    ref_logits, rows, ref_events, _ = sref.infer(path, x)
    em = M.EncryptedModel(spec, schedule=schedule, security=security)
    if security:
        assert em.security["meets_128"] and em.security["log2_qp"] <= 1747
    rec = em.ctx.attach_recorder()
    r = em.infer(x)
    ev = [(e.kind, e.value) for e in rec.snapshot()]
    em.ctx.detach_recorder()
    # every bootstrap, including those placed inside residual bodies (the ledger
    # lists top-level rows only)
    assert em.n_boot == sum(1 for e in ref_events if e[0] == "bootstrap")
    assert sum(1 for e in ev if e[0] == "bootstrap") == em.n_boot
    assert [(a[0], a[2], a[3]) for a in r.ledger] == [(b[0], b[1], b[2]) for b in rows]
    if schedule == "reference":
        assert sorted(ev) == sorted(ref_events)
    else:  # same values and levels; fewer full key switches (one ModUp/ModDown per rotate-and-sum)
        assert em.ctx.stats()["ntt_limbs"] > 0
    err = float(np.abs(r.logits - ref_logits).max())
    assert err < 1e-3, f"max abs logit error {err}"
    assert int(np.argmax(r.logits)) == int(np.argmax(ref_logits))
    return err


@pytest.mark.parametrize("schedule", ["reference", "fast"])
def test_lenet5_small_ring_with_bootstrapping(schedule):
    """LeNet-5 (BASELINE configs[2] architecture) on a 2^13 ring, depth budget 12:
    five standard-placement bootstraps."""
    spec = M.lenet5(ring=8192, depth_budget=12)
    x = np.random.default_rng(3002).uniform(0, 1, (1, 28, 28))
    _compare(spec, x, schedule)


def test_lenet5_config2_ring_depth25():
    """LeNet-5 at BASELINE configs[2]: N = 2^15 (16384 slots), the reference's
    preset depth budget 25 (backend.cpp:61-76), N(0, 0.1^2) weights, beta = 8
    (models/lenet5.json relu scale), seeded U[0,1] input; bootstraps placed as
    the reference places them."""
    spec = M.lenet5(ring=32768, depth_budget=25)
    x = np.random.default_rng(3001).uniform(0, 1, (1, 28, 28))
    _compare(spec, x, "fast")


@pytest.mark.parametrize("schedule,security", [("reference", 0), ("fast", 0), ("fast", 128)])
def test_resnet20_full_ring_with_bootstrapping(schedule, security):
    """ResNet-20 (BASELINE configs[3]): N = 2^16, depth budget 12 -> 19 bootstraps,
    He-normal weights, calibrated frozen ReLU scales (beta = 8 diverges,
    SURVEY.md section 0 item 6), per-channel normalised U[0,1] input."""
    def norm(x):
        return (x - 0.5) / 0.2887

    spec = M.resnet20(ring=65536, depth_budget=12)
    cal = [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)]
    spec = M.calibrate_relu_scales(spec, cal)
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
    _compare(spec, x, schedule, security)


def test_resnet20_reference_preset_depth25():
    """ResNet-20 at the reference's own preset depth budget (25, backend.cpp:61-76) on the
    BASELINE ring N = 2^16: 18 bootstraps, fast schedule."""
    def norm(x):
        return (x - 0.5) / 0.2887

    spec = M.resnet20(ring=65536, depth_budget=25)
    cal = [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)]
    spec = M.calibrate_relu_scales(spec, cal)
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
    _compare(spec, x, "fast")


@pytest.mark.parametrize("name,shape", [("lenet5", (1, 28, 28)), ("resnet20", (3, 32, 32))])
def test_reference_model_files_end_to_end(name, shape):
    """The reference's own models/lenet5.json (preset "lenet5": N=2^14) and
    models/resnet20.json (preset "large": N=2^15), depth budget 25, seeded CSV
    weights (tests/model_files.py), ReLU scales calibrated as the reference's
    calibrate step does, loaded by the model runtime and run encrypted."""
    from model_files import materialize
    spec = M.load_spec(materialize(name, tempfile.mkdtemp(), seed=9))
    if name == "resnet20":
        def prep(x):
            return (x - 0.5) / 0.2887
    else:
        def prep(x):
            return x
    cal = [prep(np.random.default_rng(500 + i).uniform(0, 1, shape)) for i in range(4)]
    spec = M.calibrate_relu_scales(spec, cal)
    _compare(spec, prep(np.random.default_rng(501).uniform(0, 1, shape)), "fast")


def test_batchnorm_explicit_bootstraps_end_to_end():
    """A reference-format spec with a batchnorm folded into its conv and
    explicitly placed bootstraps (bootstrap_policy "explicit")."""
    import json
    import os
    tmp = tempfile.mkdtemp()
    rng = np.random.default_rng(21)
    np.savetxt(os.path.join(tmp, "c1_w.csv"), rng.normal(0, 0.3, (1, 4 * 9)), delimiter=",", fmt="%.17g")
    np.savetxt(os.path.join(tmp, "fc_w.csv"), rng.normal(0, 0.1, (3, 4 * 36)), delimiter=",", fmt="%.17g")
    spec = {"name": "bnnet", "context": {"ring_dimension": 8192, "slot_count": 4096, "depth_budget": 9},
            "bootstrap_policy": "explicit", "input": {"channels": 1, "width": 8},
            "layers": [{"type": "conv", "name": "c1", "out_channels": 4, "kernel": 3, "weights": "c1_w.csv"},
                       {"type": "batchnorm", "gamma": [1.1, 0.9, 1.0, 1.2], "beta": [0.0, 0.1, -0.1, 0.05],
                        "mean": [0.01, -0.02, 0.03, 0.0], "var": [1.0, 0.8, 1.3, 0.9]},
                       {"type": "relu", "name": "r1", "degree": 7, "scale": 4.0}, {"type": "bootstrap"},
                       {"type": "relu", "name": "r2", "degree": 27, "scale": 4.0}, {"type": "bootstrap"},
                       {"type": "fc", "name": "fc", "outputs": 3, "weights": "fc_w.csv"}]}
    path = os.path.join(tmp, "bnnet.json")
    json.dump(spec, open(path, "w"))
    x = np.random.default_rng(22).uniform(0, 1, (1, 8, 8))
    ref_logits, rows, ref_events, _ = sref.infer(path, x)
    em = M.EncryptedModel(M.load_spec(path), security=0)
    r = em.infer(x)
    assert [(a[0], a[2], a[3]) for a in r.ledger] == [(b[0], b[1], b[2]) for b in rows]
    assert float(np.abs(r.logits - ref_logits).max()) < 1e-3


def test_lenet5_no_bootstrap_deep_budget():
    """Depth budget deep enough that the ledger needs no bootstrap except the
    standard placements (policy auto)."""
    spec = M.lenet5(ring=8192, depth_budget=25)
    x = np.random.default_rng(3003).uniform(0, 1, (1, 28, 28))
    _compare(spec, x)


def test_layer_keys_reference_schedule_equal_reference_derive():
    """Under the reference rotation schedule the engine's probed per-layer key
    sets equal the reference's derive_* sets (BuiltModel::layer_keys,
    model_spec.cpp:944-950) for its own models/lenet5.json: same indices, same
    use counts, same ends_block flags."""
    from model_files import materialize
    path = materialize("lenet5", tempfile.mkdtemp(), seed=4)
    em = M.EncryptedModel(M.load_spec(path), schedule="reference", security=0)
    ours = em.layer_keys()
    want = sref.layer_keys(path)
    assert [(lk.keys.usage, lk.ends_block) for lk in ours] == [(u, e) for u, e in want]


@pytest.mark.parametrize("name", ["lenet5", "resnet20"])
def test_block_key_mode_residency(name):
    """key_mode "block" (model_run.cpp:150): the keys of plan_blocks' block b are
    made resident before it and dropped after it when the next block does not
    use them.  Same logits bit for bit (dropped keys regenerate identically),
    the recorded trace replays cleanly against the plan, and the peak resident
    key memory is below the preload run's.  Same logits within encryption noise
    (every inference encrypts afresh)."""
    from model_files import materialize
    spec = M.load_spec(materialize(name, tempfile.mkdtemp(), seed=5))
    shape = (spec.input_channels, spec.input_width, spec.input_width)

    def prep(x):
        return (x - 0.5) / 0.2887 if name == "resnet20" else x

    spec = M.calibrate_relu_scales(spec, [prep(np.random.default_rng(600 + i).uniform(0, 1, shape))
                                          for i in range(3)])
    x = prep(np.random.default_rng(6).uniform(0, 1, shape))
    em = M.EncryptedModel(spec, security=0)
    pre = em.infer(x, verify_keys=True)
    assert pre.trace_check.ok() and pre.trace_check.rotations_checked > 0
    preload_bytes = em.ctx.key_bytes()
    blk = em.infer(x, key_mode="block", verify_keys=True)
    assert blk.trace_check.ok(), blk.trace_check.violations[:3]
    assert np.abs(blk.logits - pre.logits).max() < 1e-3
    assert len(blk.plan.blocks) > 1 and blk.key_residency["dropped"] > 0
    assert blk.key_residency["peak_key_bytes"] < preload_bytes
    est = M.keyplan.estimate_memory(blk.plan, em.memory_model())
    assert est.peak_bytes < est.preload_bytes


def test_block_key_mode_streamed_from_host():
    """key_mode "block" with the keys streamed from pinned host memory (packed
    wire format, upload stream) instead of regenerated on the device: no key is
    generated during the inference, every block's missing keys are uploaded, the
    trace replays cleanly against the plan, and the logits match the reference."""
    from model_files import materialize
    path = materialize("lenet5", tempfile.mkdtemp(), seed=5)
    spec = M.load_spec(path)
    spec = M.calibrate_relu_scales(spec, [np.random.default_rng(600 + i).uniform(0, 1, (1, 28, 28))
                                          for i in range(3)])
    x = np.random.default_rng(6).uniform(0, 1, (1, 28, 28))
    em = M.EncryptedModel(spec, security=0)
    em.enable_key_streaming()
    for _ in range(2):
        r = em.infer(x, key_mode="block", verify_keys=True)
        assert r.trace_check.ok() and r.key_residency["generated"] == 0
        assert r.key_residency["uploaded"] > 0
        assert r.key_residency["uploaded_bytes"] == r.key_residency["uploaded"] * em.ctx.key_packed_words() * 8
    ref_logits, _, _, _ = sref.infer(spec.write(tempfile.mkdtemp()), x)
    assert float(np.abs(r.logits - ref_logits).max()) < 1e-3


def test_run_report_json_matches_reference_layout():
    """RunReport / to_json (model_run.cpp:407-492): same top-level keys and nested
    layout as the reference's report, the logits equal to infer()'s within noise,
    deltas against the float true-ReLU reference, clean trace check."""
    import json
    spec = M.lenet5(ring=8192, depth_budget=12)
    x = np.random.default_rng(3002).uniform(0, 1, (1, 28, 28))
    em = M.EncryptedModel(spec, security=0)
    rep = M.run_with_report(em, x, key_mode="block")
    j = json.loads(rep.to_json())
    ref_keys = {"model", "kernels", "logits", "reference_logits", "deltas", "max_abs_delta", "argmax",
                "reference_argmax", "argmax_match", "rotations", "wall_ms", "ledger", "plan", "trace_check",
                "memory", "notes"}
    assert ref_keys <= set(j) and {"security", "engine"} <= set(j)
    assert set(j["ledger"][0]) == {"layer", "declared_levels", "level_in", "level_out", "bootstrap"}
    assert set(j["plan"]) == {"blocks", "total_keys", "peak_resident_keys", "residency"}
    assert set(j["trace_check"]) == {"ok", "violations", "unused_keys"} and j["trace_check"]["ok"]
    assert set(j["memory"]) == {"total_keys", "resident_keys", "preload_bytes", "peak_bytes", "assumptions"}
    assert len(j["deltas"]) == 10 and abs(j["max_abs_delta"] - max(j["deltas"])) < 1e-15
    assert j["rotations"] > 0 and len(j["plan"]["blocks"]) >= 2
    ref_logits, _, _, _ = sref.infer(spec.write(tempfile.mkdtemp()), x)
    assert float(np.abs(np.asarray(j["logits"]) - ref_logits).max()) < 1e-3


def test_vgg16_paper_widths_128bit():
    """VGG-16 (BASELINE configs[4]) at the FHEON paper's widths (PAPER.md:844-865,
    model.vgg16_paper) on the 128-bit N = 2^16 chain: thirteen 3x3 convs, five
    poolings, three FC layers, bootstraps placed as the reference places them;
    decrypted logits within 1e-3 of the reference's infer()."""
    def norm(x):
        return (x - 0.5) / 0.2887

    cal = [norm(np.random.default_rng(5002 + i).uniform(0, 1, (3, 32, 32))) for i in range(4)]
    spec = M.calibrate_relu_scales(M.vgg16_paper(ring=65536, depth_budget=11), cal)
    _compare(spec, norm(np.random.default_rng(5001).uniform(0, 1, (3, 32, 32))), "fast", 128)


def test_forward_batch_bit_identical_to_forward():
    """forward_batch (images in lockstep, bootstraps through bootstrap_many) yields,
    per image, the very ciphertext words of forward(): LeNet-5 on a 2^13 ring with
    five bootstraps, three images; and the bootstrap count scales with the batch."""
    spec = M.lenet5(ring=8192, depth_budget=12)
    em = M.EncryptedModel(spec, security=0)
    xs = [np.random.default_rng(3100 + i).uniform(0, 1, (1, 28, 28)) for i in range(3)]
    vs = [em.encrypt_input(x) for x in xs]  # ciphertexts are immutable: both paths read the same inputs
    singles = [em.forward(v) for v in vs]
    rec = em.ctx.attach_recorder()
    many = em.forward_batch(vs)
    boots = sum(1 for e in rec.snapshot() if e.kind == "bootstrap")
    em.ctx.detach_recorder()
    assert boots == 3 * em.n_boot
    for s, m in zip(singles, many):
        assert m.level() == s.level()
        assert np.array_equal(m.words(), s.words())
    m = em.output_count()
    for x, lg, s in zip(xs, em.infer_batch(xs), singles):
        assert np.abs(lg - s.slots()[:m]).max() < 1e-5
