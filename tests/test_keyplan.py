"""Key planning (paper_2510_03996_b200/keyplan.py) against the reference's own
planner (proj/src/keyplan.cpp:280-454, through oracle/_ref): block splitting,
explicit ranges and their errors, trace replay, ends_block flags; plus the
engine's corrected key-size model.  CPU only (the GPU probe / residency tests
live in tests/test_gpu_models.py)."""
import tempfile

import numpy as np
import pytest

from oracle import ref as sref
from paper_2510_03996_b200 import keyplan as kp
from paper_2510_03996_b200 import model as M

pytestmark = pytest.mark.skipif(not sref.available(), reason="reference oracle not built")


def _ours(ref_layers):
    return [kp.LayerKeys(f"L{i}", kp.KeySet(dict(u)), e) for i, (u, e) in enumerate(ref_layers)]


def _summary(plan, check=None):
    out = ([(b.first_layer, b.last_layer, b.keys.size()) for b in plan.blocks], plan.union_keys.size(),
           plan.peak_resident_keys)
    if check is not None:
        out += (len(check.violations), len(check.unused_keys), check.rotations_checked)
    return out


@pytest.fixture(scope="module", params=["lenet5", "resnet20"])
def spec_layers(request):
    from model_files import materialize
    path = materialize(request.param, tempfile.mkdtemp(), seed=3)
    return path, sref.layer_keys(path)


def test_plans_match_reference(spec_layers):
    path, rl = spec_layers
    ours = _ours(rl)
    for mode, fn in ((0, kp.plan_single_block), (1, kp.plan_blocks)):
        want = sref.plan(mode, rl)
        assert _summary(fn(ours)) == want[:3]
    n = len(rl)
    ranges = [(0, n // 3), (n // 3 + 1, n - 2), (n - 1, n - 1)]
    assert _summary(kp.plan_blocks(ours, ranges)) == sref.plan(2, rl, ranges)[:3]


def test_ends_block_matches_reference(spec_layers):
    path, rl = spec_layers
    layers = M.build(M.load_spec(path))
    assert [M.ends_block(b) for b in layers] == [e for _, e in rl]


@pytest.mark.parametrize("ranges", [[(1, 3)], [(0, 2), (4, 5)], [(0, 1)], [(0, 3), (3, 5)]])
def test_bad_ranges_raise_like_reference(spec_layers, ranges):
    _, rl = spec_layers
    with pytest.raises(sref.RefError):
        sref.plan(2, rl, ranges)
    with pytest.raises(Exception, match="block ranges"):
        kp.plan_blocks(_ours(rl), ranges)


def test_verify_trace_matches_reference(spec_layers):
    """A replay with in-plan rotations, an out-of-block rotation, a rotation
    before any marker and a layer past the plan: same violation / unused counts."""
    _, rl = spec_layers
    ours = _ours(rl)
    plan = kp.plan_blocks(ours)
    ev = [(0, 7)]  # before any marker
    for i, (u, _) in enumerate(rl):
        ev.append((4, i))
        keys = sorted(u)
        for k in keys[: max(1, len(keys) // 2)] if keys else []:
            ev.append((0, k))
        if i == len(rl) // 2:
            ev.append((0, 123457))  # not resident anywhere
        ev.append((1, 3))
    ev += [(4, len(rl) + 5), (0, 1)]  # uncovered layer
    events = [kp.TraceEvent("rotation" if k == 0 else "marker" if k == 4 else "mult_plain", v,
                            f"layer:{v}:x" if k == 4 else "") for k, v in ev]
    chk = kp.verify_trace(plan, events)
    assert _summary(plan, chk) == sref.plan(1, rl, (), ev)
    assert not chk.ok()


def test_memory_models():
    m = kp.MemoryModel.for_engine(1 << 16, 24, 8, 3, fixed_keys=2)
    assert m.bytes_per_key == 3 * 2 * 32 * (1 << 16) * 8 == 96 << 20
    r = kp.MemoryModel.reference_model(1 << 16, 23, 3)
    assert r.bytes_per_key == 2 * 3 * (1 << 16) * 25 * 8  # keyplan.cpp:424-439
    plan = kp.plan_blocks([kp.LayerKeys("a", kp.KeySet({1: 2, 2: 1}), True), kp.LayerKeys("b", kp.KeySet({4: 1}))])
    est = kp.estimate_memory(plan, m)
    assert (est.total_keys, est.resident_keys) == (3, 2)
    assert est.preload_bytes == 5 * m.bytes_per_key and est.peak_bytes == 4 * m.bytes_per_key
