"""CPU: the model runtime reads the reference's model-spec format
(proj/models/README.md, model_spec.cpp:117-904) -- the reference's own
models/lenet5.json and models/resnet20.json with seeded CSV weights, batchnorm
folding, explicit bootstrap placement, the build-time checks -- and builds
the same model as the reference: same bootstrap placement, same per-layer
ledger as the reference's infer() report (oracle/_ref, run on the CPU)."""
import json
import os
import tempfile

import numpy as np
import pytest

import paper_2510_03996_b200 as fh
from paper_2510_03996_b200 import model as M
from oracle import ref as sref
from model_files import materialize

needs_ref = pytest.mark.skipif(not sref.available(), reason="oracle/_ref not built")


def _walk_equal(a, b):
    for x, y in zip(a, b):
        assert (x.type, x.name) == (y.type, y.name)
        for u, v in ((x.weights, y.weights), (x.bias, y.bias)):
            assert (u is None) == (v is None) and (u is None or np.array_equal(u, v))
        _walk_equal(x.body, y.body)
        _walk_equal(x.downsample, y.downsample)


@pytest.mark.parametrize("depth", [12, 25])
def test_write_load_roundtrip(depth):
    for spec in (M.lenet5(ring=32768, depth_budget=depth), M.resnet20(ring=65536, depth_budget=depth)):
        s2 = M.load_spec(spec.write(tempfile.mkdtemp()))
        assert (s2.ring_dimension, s2.slot_count, s2.depth_budget) == (spec.ring_dimension, spec.slot_count, depth)
        _walk_equal(spec.layers, s2.layers)
        assert M.count_bootstraps(M.build(spec)) == M.count_bootstraps(M.build(s2))


@needs_ref
@pytest.mark.parametrize("name,shape,boots", [("lenet5", (1, 28, 28), 3), ("resnet20", (3, 32, 32), 18)])
def test_reference_model_files_build_like_the_reference(name, shape, boots):
    """models/lenet5.json (preset "lenet5") and models/resnet20.json (preset "large"),
    depth budget 25: same bootstraps and ledger rows as the reference's infer()."""
    path = materialize(name, tempfile.mkdtemp(), seed=5)
    spec = M.load_spec(path)
    layers = M.build(spec)
    assert M.count_bootstraps(layers) == boots
    x = np.random.default_rng(6).uniform(0, 1, shape)
    _, rows, events, _ = sref.infer(path, x)
    assert [tuple(r) for r in M.ledger_rows(layers, spec.depth_budget)] == [tuple(r) for r in rows]
    assert sum(1 for e in events if e[0] == "bootstrap") == boots


def _bn_spec(tmp, explicit=False, bn_inline=True):
    rng = np.random.default_rng(11)
    w = rng.normal(0, 0.3, (4, 1, 3, 3))
    np.savetxt(os.path.join(tmp, "c1_w.csv"), w.reshape(1, -1), delimiter=",", fmt="%.17g")
    np.savetxt(os.path.join(tmp, "c1_b.csv"), rng.normal(0, 0.1, (1, 4)), delimiter=",", fmt="%.17g")
    fcw = rng.normal(0, 0.1, (3, 4 * 6 * 6))
    np.savetxt(os.path.join(tmp, "fc_w.csv"), fcw, delimiter=",", fmt="%.17g")
    bn = {"type": "batchnorm", "name": "bn1", "gamma": [1.1, 0.9, 1.0, 1.2], "beta": [0.0, 0.1, -0.1, 0.05],
          "mean": [0.01, -0.02, 0.03, 0.0], "var": [1.0, 0.8, 1.3, 0.9], "epsilon": 1e-5}
    if not bn_inline:
        np.savetxt(os.path.join(tmp, "bn_var.csv"), np.array([[1.0, 0.8, 1.3, 0.9]]), delimiter=",")
        bn["var"] = "bn_var.csv"
    layers = [{"type": "conv", "name": "c1", "out_channels": 4, "kernel": 3, "weights": "c1_w.csv", "bias": "c1_b.csv"},
              bn, {"type": "relu", "name": "r1", "degree": 7}]
    boot = [{"type": "bootstrap"}] if explicit else []  # default names bootstrap_<index>
    layers += boot + [{"type": "relu", "name": "r2", "degree": 27}] + boot + \
        [{"type": "relu", "name": "r3", "degree": 27}, {"type": "fc", "name": "fc", "outputs": 3, "weights": "fc_w.csv"}]
    spec = {"name": "bnnet", "context": {"ring_dimension": 4096, "slot_count": 2048, "depth_budget": 9},
            "bootstrap_policy": "explicit" if explicit else "auto", "input": {"channels": 1, "width": 8},
            "layers": layers}
    path = os.path.join(tmp, "bnnet.json")
    json.dump(spec, open(path, "w"))
    return path, w, bn


@pytest.mark.parametrize("inline", [True, False])
def test_batchnorm_folds_into_the_convolution(inline):
    tmp = tempfile.mkdtemp()
    path, w, bn = _bn_spec(tmp, bn_inline=inline)
    spec = M.load_spec(path)
    assert [L.type for L in spec.layers] == ["conv", "relu", "relu", "relu", "fc"]
    assert [L.name for L in spec.layers] == ["c1", "r1", "r2", "r3", "fc"]
    s = np.array(bn["gamma"]) / np.sqrt(np.array([1.0, 0.8, 1.3, 0.9]) + bn["epsilon"])
    assert np.allclose(spec.layers[0].weights, w * s[:, None, None, None], rtol=0, atol=1e-15)
    b = np.loadtxt(os.path.join(tmp, "c1_b.csv"), delimiter=",")
    assert np.allclose(spec.layers[0].bias, s * (b - np.array(bn["mean"])) + np.array(bn["beta"]), atol=1e-15)


@needs_ref
def test_explicit_policy_holds_or_fails_like_the_reference():
    tmp = tempfile.mkdtemp()
    ok, _, _ = _bn_spec(tmp, explicit=True)
    spec = M.load_spec(ok)
    layers = M.build(spec)
    assert M.count_bootstraps(layers) == 2
    x = np.random.default_rng(1).uniform(0, 1, (1, 8, 8))
    _, rows, _, _ = sref.infer(ok, x)
    assert [tuple(r) for r in M.ledger_rows(layers, spec.depth_budget)] == [tuple(r) for r in rows]
    bad, _, _ = _bn_spec(tempfile.mkdtemp(), explicit=False)
    d = json.load(open(bad))
    d["bootstrap_policy"] = "explicit"
    json.dump(d, open(bad, "w"))
    with pytest.raises(fh.ModelError) as e:
        M.build(M.load_spec(bad))
    assert "explicit bootstrap placement" in str(e.value)
    with pytest.raises(sref.RefError) as r:
        sref.infer(bad, x)
    assert r.value.category == e.value.category == 2


@needs_ref
@pytest.mark.parametrize("mutate,fragment", [
    (lambda d: d["layers"].append({"type": "dropout"}), "unknown layer type"),
    (lambda d: d["layers"][0].update(kernel=4, stride=3), "layer 'c1'"),
    (lambda d: d["layers"][0].update(weights="missing.csv"), "cannot open"),
    (lambda d: d["layers"][-1].update(inputs=7), "declares 7 inputs"),
    (lambda d: d["layers"].insert(0, {"type": "batchnorm", "gamma": [1], "beta": [0], "mean": [0], "var": [1]}),
     "must directly follow a convolution"),
    (lambda d: d.update(bootstrap_policy="sometimes"), "bootstrap_policy"),
])
def test_invalid_specs_fail_like_the_reference(mutate, fragment):
    tmp = tempfile.mkdtemp()
    path, _, _ = _bn_spec(tmp)
    d = json.load(open(path))
    mutate(d)
    json.dump(d, open(path, "w"))
    x = np.random.default_rng(1).uniform(0, 1, (1, 8, 8))
    with pytest.raises(fh.ModelError) as e:
        M.build(M.load_spec(path))
    assert fragment in str(e.value)
    with pytest.raises(sref.RefError) as r:
        sref.infer(path, x)
    assert r.value.category == e.value.category


@needs_ref
def test_vgg16_does_not_fit_32768_slots_like_the_reference():
    """BASELINE configs[4] VGG-16 at N=2^16: the first block's 64x32x32 output
    needs 65536 slots; the reference's build fails with ModelError (BASELINE.md
    section 2) and so does ours, with the same message and category."""
    spec = M.vgg16(ring=65536)
    with pytest.raises(fh.ModelError) as e:
        M.build(spec)
    assert "output needs 65536 slots, context provides 32768" in str(e.value)
    path = spec.write(tempfile.mkdtemp())
    with pytest.raises(sref.RefError) as r:
        sref.infer(path, np.zeros((3, 32, 32)))
    assert "output needs 65536 slots, context provides 32768" in str(r.value)
    assert r.value.category == e.value.category

