"""Rotation-key planning and HBM residency.

Restates the reference's planning layer (proj/include/slotcnn/keyplan.hpp:25-150,
proj/src/keyplan.cpp:280-454): a KeySet multiset per layer, blocks of layers
whose keys must be resident together (plan_single_block / plan_blocks, split
after every layer that shrinks the grid, keyplan.cpp:330-344), replay of a trace
against a plan (verify_trace, keyplan.cpp:370-421) and memory estimates.

Two deliberate differences, both because this engine does real CKKS:

* Keys per layer are DERIVED FROM THE ENGINE, not from the reference's layer
  algebra (keyplan.cpp:120-278 derive_*): the fast rotation schedule uses
  different (fewer) rotations, so `EncryptedModel.layer_keys()` probes one
  inference and records every layer's rotation indices (the schedule depends on
  shapes only, so any input gives the same set).  Under the reference schedule
  the probe reproduces the reference's derive_* sets exactly (same trace
  multiset, tests/test_gpu_layers.py).
* MemoryModel uses the engine's true hybrid key size, dnum x 2 x (L + K) x N x 8
  bytes, instead of the reference's
  2 x digits x N x (depth + 2) x 8 (keyplan.cpp:424-439), which undercounts the
  special primes and the full chain; bootstrapping and relinearisation keys are
  the fixed overhead (the reference carries bootstrapping as an opaque flag).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from .api import ShapeError

NPOS = -1


@dataclass
class KeySet:
    """Rotation index -> planned number of uses (keyplan.hpp:27-41); index 0 never appears."""
    usage: Dict[int, int] = field(default_factory=dict)

    def add(self, index: int, count: int = 1):
        if index != 0 and count > 0:
            self.usage[int(index)] = self.usage.get(int(index), 0) + int(count)

    def merge(self, other: "KeySet"):
        for k, v in other.usage.items():
            self.add(k, v)

    def merge_scaled(self, other: "KeySet", times: int):
        for k, v in other.usage.items():
            self.add(k, v * times)

    def indices(self) -> List[int]:
        return sorted(self.usage)

    def size(self) -> int:
        return len(self.usage)

    def contains(self, index: int) -> bool:
        return int(index) in self.usage

    def total_uses(self) -> int:
        return sum(self.usage.values())


@dataclass
class LayerKeys:
    name: str
    keys: KeySet
    ends_block: bool = False  # the layer shrinks the grid (model_spec.cpp:521,555,577,708)


@dataclass
class Block:
    first_layer: int
    last_layer: int  # inclusive
    keys: KeySet = field(default_factory=KeySet)


@dataclass
class BlockPlan:
    blocks: List[Block] = field(default_factory=list)
    union_keys: KeySet = field(default_factory=KeySet)
    peak_resident_keys: int = 0
    residency_events: List[str] = field(default_factory=list)

    def block_of_layer(self, layer: int) -> int:
        for b, blk in enumerate(self.blocks):
            if blk.first_layer <= layer <= blk.last_layer:
                return b
        return NPOS


def _finalize(layers: Sequence[LayerKeys], blocks: List[Block]) -> BlockPlan:
    """finalize_plan (keyplan.cpp:284-306)."""
    plan = BlockPlan(blocks=blocks)
    for blk in plan.blocks:
        for i in range(blk.first_layer, blk.last_layer + 1):
            blk.keys.merge(layers[i].keys)
        plan.union_keys.merge(blk.keys)
        plan.peak_resident_keys = max(plan.peak_resident_keys, blk.keys.size())
    for b, blk in enumerate(plan.blocks):
        plan.residency_events.append(
            f"{'load block ' if b == 0 else 'swap to block '}{b} ({blk.keys.size()} rotation keys) before layer "
            f"{blk.first_layer} ({layers[blk.first_layer].name})")
    return plan


def plan_single_block(layers: Sequence[LayerKeys]) -> BlockPlan:
    """Everything resident for the whole run (keyplan.cpp:319-328)."""
    if not layers:
        return BlockPlan()
    return _finalize(layers, [Block(0, len(layers) - 1)])


def plan_blocks(layers: Sequence[LayerKeys],
                ranges: Optional[Sequence[Tuple[int, int]]] = None) -> BlockPlan:
    """Blocks split after every ends_block layer (keyplan.cpp:330-344), or explicit
    [first, last] ranges that must tile the layers in order (keyplan.cpp:346-368)."""
    if not layers:
        return BlockPlan()
    blocks: List[Block] = []
    if ranges is None:
        first = 0
        for i, lk in enumerate(layers):
            boundary = lk.ends_block and i + 1 < len(layers)
            if boundary or i + 1 == len(layers):
                blocks.append(Block(first, i))
                first = i + 1
        return _finalize(layers, blocks)
    expect = 0
    for first, last in ranges:
        if first != expect or last < first or last >= len(layers):
            raise ShapeError("block ranges must tile the layer list in order without gaps", 2)
        blocks.append(Block(first, last))
        expect = last + 1
    if expect != len(layers):
        raise ShapeError("block ranges leave trailing layers unassigned", 2)
    return _finalize(layers, blocks)


@dataclass
class TraceEvent:
    kind: str            # "rotation", "mult_plain", "mult_cipher", "bootstrap", "marker"
    value: int = 0
    label: str = ""


@dataclass
class Violation:
    event_index: int
    rotation_index: int
    layer: int
    reason: str


@dataclass
class TraceCheck:
    violations: List[Violation] = field(default_factory=list)
    unused_keys: List[int] = field(default_factory=list)
    rotations_checked: int = 0

    def ok(self) -> bool:
        return not self.violations


def verify_trace(plan: BlockPlan, events: Sequence[TraceEvent]) -> TraceCheck:
    """Every rotation must use an index resident in the block of the layer
    executing at that point; layer boundaries are "layer:<index>:<name>"
    markers (keyplan.cpp:370-421)."""
    check = TraceCheck()
    observed: Dict[int, int] = {}
    current = NPOS
    for idx, e in enumerate(events):
        if e.kind == "marker":
            if e.label.startswith("layer:"):
                try:
                    current = int(e.label[6:].split(":", 1)[0])
                except ValueError:
                    check.violations.append(Violation(idx, 0, NPOS, "unparseable layer marker: " + e.label))
            continue
        if e.kind != "rotation":
            continue
        check.rotations_checked += 1
        observed[e.value] = observed.get(e.value, 0) + 1
        if current == NPOS:
            check.violations.append(Violation(idx, e.value, NPOS, "rotation issued before any layer marker"))
            continue
        b = plan.block_of_layer(current)
        if b == NPOS:
            check.violations.append(Violation(idx, e.value, current, "layer is not covered by any block"))
            continue
        if not plan.blocks[b].keys.contains(e.value):
            check.violations.append(Violation(idx, e.value, current,
                                              f"rotation index {e.value} is not resident in block {b}"))
    check.unused_keys = [i for i in plan.union_keys.indices() if i not in observed]
    return check


@dataclass
class MemoryModel:
    bytes_per_key: int = 0
    fixed_overhead_bytes: int = 0
    assumptions: str = ""

    @staticmethod
    def for_engine(ring_dimension: int, limbs: int, special_limbs: int, dnum: int,
                   fixed_keys: int = 0) -> "MemoryModel":
        """The engine's evaluation-key layout [dnum][2][L+K][N] u64;
        `fixed_keys` (relinearisation, conjugation, bootstrapping rotations) stay resident."""
        b = dnum * 2 * (limbs + special_limbs) * ring_dimension * 8
        return MemoryModel(b, fixed_keys * b,
                           f"bytes_per_key = {dnum} digits x 2 ring elements x {limbs + special_limbs} limbs "
                           f"(L={limbs} + K={special_limbs}) x {ring_dimension} coefficients x 8 bytes; "
                           f"{fixed_keys} relinearisation/bootstrapping keys resident throughout")

    @staticmethod
    def reference_model(ring_dimension: int, depth_budget: int, key_switch_digits: int) -> "MemoryModel":
        """The reference's estimate (keyplan.cpp:424-439), kept for comparison."""
        limbs = depth_budget + 2
        return MemoryModel(2 * key_switch_digits * ring_dimension * limbs * 8, 0,
                           f"bytes_per_key = 2 ring elements x {key_switch_digits} decomposition digits x "
                           f"{limbs} residue limbs x {ring_dimension} coefficients x 8 bytes")


@dataclass
class MemoryEstimate:
    total_keys: int = 0
    resident_keys: int = 0
    preload_bytes: int = 0
    peak_bytes: int = 0
    assumptions: str = ""


def estimate_memory(plan: BlockPlan, model: MemoryModel) -> MemoryEstimate:
    """keyplan.cpp:441-452."""
    est = MemoryEstimate(total_keys=plan.union_keys.size(), resident_keys=plan.peak_resident_keys,
                         assumptions=model.assumptions)
    est.preload_bytes = est.total_keys * model.bytes_per_key + model.fixed_overhead_bytes
    est.peak_bytes = est.resident_keys * model.bytes_per_key + model.fixed_overhead_bytes
    return est
