"""Model runtime over the B200 engine.

Host-side mirror of the reference's model runtime:
  spec        proj/src/model_spec.cpp:117-272  (JSON schema of models/README.md)
  build       proj/src/model_spec.cpp:456-904  (shape flow, declared depth costs,
              standard bootstrap placement :746-776, ledger repair :789-851)
  infer       proj/src/model_run.cpp:100-159   (per-layer ledger assertion)
  calibrate   proj/src/model_run.cpp:364-403   (ReLU range bounds, safety 1.25)
Every layer runs as one C-ABI call into the sm_100a engine; this module only
orchestrates (shapes, levels, placement) -- no arithmetic happens here.

Model builders `lenet5()` / `resnet20()` construct the BASELINE configs[2] /
configs[3] architectures with seeded random weights (the reference ships no
weights and the container has no datasets); `ModelSpec.write()` emits the
reference's JSON + CSV format so the same model runs through oracle/_ref.
"""
from __future__ import annotations

import copy
import json
import math
import os
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import api as fh
from . import keyplan


# ----------------------------------------------------------------- spec
@dataclass
class Layer:
    type: str
    name: str
    params: Dict = field(default_factory=dict)
    weights: Optional[np.ndarray] = None
    bias: Optional[np.ndarray] = None
    body: List["Layer"] = field(default_factory=list)
    downsample: List["Layer"] = field(default_factory=list)


@dataclass
class ModelSpec:
    name: str
    ring_dimension: int
    slot_count: int
    depth_budget: int
    input_channels: int
    input_width: int
    layers: List[Layer]
    bootstrap_policy: str = "auto"
    weight_mode: str = "preload"  # "lazy": no resident weight plaintexts (model.hpp:46-48)

    def write(self, directory: str) -> str:
        """Reference JSON spec + CSV weights (models/README.md format)."""
        os.makedirs(directory, exist_ok=True)

        def enc(L: Layer) -> Dict:
            d = {"type": L.type, "name": L.name}
            d.update(L.params)
            if L.weights is not None:
                fn = f"{L.name}_weights.csv"
                np.savetxt(os.path.join(directory, fn), L.weights.reshape(1, -1), delimiter=",", fmt="%.17g")
                d["weights"] = fn
            if L.bias is not None:
                fn = f"{L.name}_bias.csv"
                np.savetxt(os.path.join(directory, fn), L.bias.reshape(1, -1), delimiter=",", fmt="%.17g")
                d["bias"] = fn
            if L.type == "residual":
                d["layers"] = [enc(b) for b in L.body]
                if L.downsample:
                    d["downsample"] = enc(L.downsample[0])  # a single conv object
            return d

        spec = {"name": self.name,
                "context": {"ring_dimension": self.ring_dimension, "slot_count": self.slot_count,
                            "depth_budget": self.depth_budget},
                "weight_mode": self.weight_mode, "bootstrap_policy": self.bootstrap_policy,
                "input": {"channels": self.input_channels, "width": self.input_width},
                "layers": [enc(L) for L in self.layers]}
        path = os.path.join(directory, f"{self.name}.json")
        with open(path, "w") as f:
            json.dump(spec, f, indent=1)
        return path


# ----------------------------------------------------------------- spec files
_PRESETS = {"lenet5": (16384, 8192, 25), "large": (32768, 16384, 25)}  # backend.cpp:61-76


def _fail(msg: str):
    raise fh.ModelError(msg, 2)


def _size(j: Dict, key: str, where: str, default=None) -> int:
    if key not in j:
        if default is None:
            _fail(f'{where}: missing required field "{key}"')
        return default
    v = j[key]
    if isinstance(v, bool) or not isinstance(v, int) or v < 0:
        _fail(f'{where}: field "{key}" must be a non-negative integer')
    return v


def _csv_values(path: str, expected: int, what: str) -> np.ndarray:
    """load_csv_values (model_spec.cpp:293-337): comma/newline separated numbers,
    blank cells skipped, exact count required."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        _fail(f"{what}: cannot open {path}")
    out = []
    for row, line in enumerate(text.splitlines(), start=1):
        for col, tok in enumerate(line.split(","), start=1):
            tok = tok.strip()
            if not tok:
                continue
            try:
                out.append(float(tok))
            except ValueError:
                _fail(f'{what}: {path} row {row} column {col}: cannot parse "{tok}" as a number')
    if len(out) != expected:
        _fail(f"{what}: {path}: expected {expected} values, found {len(out)}")
    return np.array(out, np.float64)


def _parse_layer(j, index: int, scope: str) -> Layer:
    """parse_layer (model_spec.cpp:133-207)."""
    where = f"{scope}layers[{index}]"
    if not isinstance(j, dict) or not isinstance(j.get("type"), str):
        _fail(f'{where}: every layer needs a string "type"')
    t = j["type"]
    name = j.get("name", f"{t}_{index}")
    p: Dict = {}
    if t == "conv":
        p["out_channels"] = _size(j, "out_channels", where)
        p["kernel"] = _size(j, "kernel", where)
        p["stride"] = _size(j, "stride", where, 1)
        p["padding"] = _size(j, "padding", where, 0)
        mode = j.get("mode", "generic")
        if mode not in ("generic", "special3x3", "grouped"):
            _fail(f'{where}: mode must be "generic", "special3x3" or "grouped", got "{mode}"')
        p["mode"] = mode
    elif t == "avg_pool":
        p["kernel"] = _size(j, "kernel", where, 2)
        p["stride"] = _size(j, "stride", where, 2)
    elif t == "whole_channel_pool":
        p["kernel"] = _size(j, "kernel", where)
    elif t == "fc":
        p["outputs"] = _size(j, "outputs", where)
        p["inputs"] = _size(j, "inputs", where, 0)
        p["merge_budget"] = _size(j, "merge_budget", where, 1)
    elif t == "relu":
        if "degree" in j:
            p["degree"] = int(j["degree"])
        if "scale" in j:
            p["scale"] = float(j["scale"])
    elif t == "batchnorm":
        for key in ("gamma", "beta", "mean", "var"):
            if key not in j:
                _fail(f'{where}: batchnorm needs field "{key}"')
            v = j[key]
            if not isinstance(v, (list, str)):
                _fail(f'{where}: "{key}" must be an array of numbers or a CSV file name')
            p[key] = v
        p["epsilon"] = float(j.get("epsilon", 1e-5))
    elif t in ("global_avg_pool", "bootstrap"):
        pass
    elif t == "residual":
        if "layers" not in j:
            _fail(f'{where}: residual units need a nested "layers" array')
        L = Layer(t, name, p, body=_parse_list(j["layers"], where + "."))
        if "downsample" in j:
            d = _parse_layer(j["downsample"], 0, where + ".downsample.")
            if d.type != "conv":
                _fail(f'{where}: "downsample" must be a conv layer')
            L.downsample = [d]
        return L
    else:
        _fail(f'{where}: unknown layer type "{t}"')
    if t in ("conv", "avg_pool"):
        sv = j.get("stride_variant", "extract")
        if sv not in ("extract", "masked"):
            _fail(f'{where}: stride_variant must be "extract" or "masked", got "{sv}"')
        p["stride_variant"] = sv
    if t in ("conv", "fc"):
        p["weights_file"] = j.get("weights", "")
        p["bias_file"] = j.get("bias", "")
    return Layer(t, name, p)


def _parse_list(j, scope: str) -> List[Layer]:
    if not isinstance(j, list) or not j:
        _fail(f'{scope}: "layers" must be a non-empty array')
    return [_parse_layer(e, i, scope) for i, e in enumerate(j)]


def _resolve_file(base: str, f: str) -> str:
    return f if os.path.isabs(f) else os.path.join(base, f)


def _load_weights(layers: List[Layer], shape, base: str) -> Tuple[List[Layer], Tuple]:
    """Read every conv / fc weight file with the flow's input sizes and fold
    batchnorm into the convolution before it (model_spec.cpp:349-406, :643-684)."""
    out: List[Layer] = []
    folded = set()
    for L in layers:
        packed, C, W, n = shape
        if L.type == "conv":
            p = L.params
            F, k, S, P = p["out_channels"], p["kernel"], p["stride"], p["padding"]
            wc = 1 if p["mode"] == "grouped" else C
            if not p.get("weights_file"):
                _fail(f"layer '{L.name}': no weights file given")
            L.weights = _csv_values(_resolve_file(base, p.pop("weights_file")), F * wc * k * k,
                                    f"layer '{L.name}' weights").reshape(F, wc, k, k)
            bf = p.pop("bias_file", "")
            L.bias = _csv_values(_resolve_file(base, bf), F, f"layer '{L.name}' bias") if bf else None
            if k == 0 or S == 0 or F == 0:
                _fail(f"layer '{L.name}': out_channels, kernel and stride must be positive")
            Wo = (W + 2 * P - k) // S + 1 if W + 2 * P >= k else 0
            shape = (True, F, Wo, 0)
        elif L.type == "batchnorm":
            if not out or out[-1].type != "conv":
                _fail(f"layer '{L.name}': batchnorm must directly follow a convolution")
            conv = out[-1]
            if conv.name in folded:
                _fail(f"layer '{L.name}': convolution '{conv.name}' already has batchnorm folded in")
            F = conv.params["out_channels"]
            vec = {}
            for key in ("gamma", "beta", "mean", "var"):
                v = L.params[key]
                vec[key] = (_csv_values(_resolve_file(base, v), F, f"layer '{L.name}' {key}") if isinstance(v, str)
                            else np.asarray(v, np.float64))
                if vec[key].size != F:
                    _fail(f"layer '{L.name}' {key}: expected {F} values, found {vec[key].size}")
            eps = L.params["epsilon"]
            if not np.all(vec["var"] + eps > 0):
                _fail(f"layer '{L.name}': variance + epsilon must be positive")
            sc = vec["gamma"] / np.sqrt(vec["var"] + eps)
            conv.weights = conv.weights * sc[:, None, None, None]
            b = conv.bias if conv.bias is not None else np.zeros(F)
            conv.bias = sc * (b - vec["mean"]) + vec["beta"]
            folded.add(conv.name)
            continue
        elif L.type == "avg_pool":
            k, S = L.params["kernel"], L.params["stride"]
            shape = (True, C, (W - k) // S + 1 if W >= k and S else 0, 0)
        elif L.type in ("global_avg_pool", "whole_channel_pool"):
            shape = (False, 0, 0, C)
        elif L.type == "fc":
            p = L.params
            have = C * W * W if packed else n
            if p["inputs"] and p["inputs"] != have:
                _fail(f"layer '{L.name}': declares {p['inputs']} inputs but receives {have}")
            m = p["outputs"]
            if not p.get("weights_file"):
                _fail(f"layer '{L.name}': no weights file given")
            L.weights = _csv_values(_resolve_file(base, p.pop("weights_file")), m * have,
                                    f"layer '{L.name}' weights").reshape(m, have)
            bf = p.pop("bias_file", "")
            L.bias = _csv_values(_resolve_file(base, bf), m, f"layer '{L.name}' bias") if bf else None
            shape = (False, 0, 0, m)
        elif L.type == "residual":
            L.body, bshape = _load_weights(L.body, shape, base)
            if L.downsample:
                L.downsample, _ = _load_weights(L.downsample, shape, base)
            shape = bshape
        out.append(L)
    return out, shape


def load_spec(path: str) -> ModelSpec:
    """ModelSpec::from_json_file (model_spec.cpp:232-272): a reference model spec
    (models/README.md schema) with its CSV weights, batchnorm folded.  The engine
    packs fully, so the context's slot_count must be ring_dimension / 2."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        _fail(f"cannot open model spec file {path}")
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        _fail(f"model spec is not valid JSON: {e}")
    base = os.path.dirname(os.path.abspath(path))
    ctx = j.get("context", {})
    if isinstance(ctx, str):
        if ctx not in _PRESETS:
            _fail(f'unknown context preset "{ctx}" (expected "lenet5" or "large")')
        ring, slots, depth = _PRESETS[ctx]
    elif isinstance(ctx, dict):
        ring = ctx.get("ring_dimension", 16384)
        slots = ctx.get("slot_count", 8192)
        depth = ctx.get("depth_budget", 10)
    else:
        _fail('"context" must be a preset name or a parameter object')
    weight_mode = j.get("weight_mode", "preload")
    if weight_mode not in ("preload", "lazy"):
        _fail(f'weight_mode must be "preload" or "lazy", got "{weight_mode}"')
    policy = j.get("bootstrap_policy", "auto")
    if policy not in ("auto", "explicit"):
        _fail(f'bootstrap_policy must be "auto" or "explicit", got "{policy}"')
    inp = j.get("input")
    if not isinstance(inp, dict):
        _fail('model spec needs an "input" object with channels and width')
    C, W = _size(inp, "channels", "input"), _size(inp, "width", "input")
    if "layers" not in j:
        _fail('model spec needs a "layers" array')
    layers = _parse_list(j["layers"], "")
    layers, _ = _load_weights(layers, (True, C, W, 0), base)
    return ModelSpec(j.get("name", "model"), ring, slots, depth, C, W, layers, policy, weight_mode)


def _conv(name, f, c, k, rng, std, stride=1, padding=0, mode="generic", bias=True):
    w = rng.normal(0.0, std, (f, c, k, k))
    b = rng.normal(0.0, std, f) if bias else None
    p = {"out_channels": f, "kernel": k}
    if stride != 1:
        p["stride"] = stride
    if padding:
        p["padding"] = padding
    if mode != "generic":
        p["mode"] = mode
    return Layer("conv", name, p, w, b)


def lenet5(seed: int = 3001, ring: int = 32768, depth_budget: int = 12, relu_scale: float = 8.0) -> ModelSpec:
    """BASELINE configs[2]: 1x28x28 input; conv 1->6 5x5, polyReLU, avgpool 2x2,
    conv 6->16 5x5, polyReLU, avgpool 2x2, FC 256->120->84->10; weights N(0, 0.1^2);
    degree-59 Chebyshev ReLU on inputs pre-scaled by 1/8."""
    rng = np.random.default_rng(seed)
    relu = lambda n: Layer("relu", n, {"degree": 59, "scale": relu_scale})  # noqa: E731

    def fc(name, m, n):
        return Layer("fc", name, {"outputs": m}, rng.normal(0, 0.1, (m, n)), rng.normal(0, 0.1, m))

    layers = [_conv("conv1", 6, 1, 5, rng, 0.1), relu("relu1"),
              Layer("avg_pool", "pool1", {"kernel": 2, "stride": 2}),
              _conv("conv2", 16, 6, 5, rng, 0.1), relu("relu2"),
              Layer("avg_pool", "pool2", {"kernel": 2, "stride": 2}),
              fc("fc1", 120, 256), relu("relu3"), fc("fc2", 84, 120), relu("relu4"), fc("fc3", 10, 84)]
    return ModelSpec("lenet5", ring, ring // 2, depth_budget, 1, 28, layers)


def resnet20(seed: int = 4001, ring: int = 65536, depth_budget: int = 12) -> ModelSpec:
    """BASELINE configs[3]: 3x32x32; 3x3 convs at 16/32/64 channels (special3x3),
    three stages of three basic blocks, 2x2/s2 downsampling (conv + projection),
    global avgpool, FC 64->10; He-normal weights, bias 0."""
    rng = np.random.default_rng(seed)

    def he(c, k):
        return math.sqrt(2.0 / (c * k * k))

    def c3(name, f, c):
        return _conv(name, f, c, 3, rng, he(c, 3), padding=1, mode="special3x3", bias=False)

    def relu(n):
        return Layer("relu", n, {"degree": 59, "scale": 8.0})

    layers = [c3("conv_in", 16, 3), relu("relu_in")]
    C = 16
    for stage, F in enumerate((16, 32, 64), start=1):
        for unit in range(1, 4):
            nm = f"unit{stage}_{unit}"
            if stage > 1 and unit == 1:
                body = [_conv(nm + "_conv1", F, C, 2, rng, he(C, 2), stride=2, bias=False), relu(nm + "_relu"),
                        c3(nm + "_conv2", F, F)]
                ds = [_conv(nm + "_proj", F, C, 2, rng, he(C, 2), stride=2, bias=False)]
            else:
                body = [c3(nm + "_conv1", F, C), relu(nm + "_relu"), c3(nm + "_conv2", F, F)]
                ds = []
            layers.append(Layer("residual", nm, {}, body=body, downsample=ds))
            layers.append(relu(nm + "_relu_out"))
            C = F
    layers.append(Layer("global_avg_pool", "pool_global"))
    layers.append(Layer("fc", "fc_out", {"outputs": 10}, rng.normal(0, math.sqrt(2.0 / 64), (10, 64)), np.zeros(10)))
    return ModelSpec("resnet20", ring, ring // 2, depth_budget, 3, 32, layers)


def vgg16(seed: int = 5001, ring: int = 65536, depth_budget: int = 25) -> ModelSpec:
    """BASELINE configs[4]: 3x32x32 input, thirteen 3x3 convs (64-64-128-128-256x3-
    512x3-512x3, pad 1), 2x2 average pooling after each block, FC 512->512->10,
    He-normal weights.  With full packing the first block's 64x32x32 output
    needs 65536 slots: at N = 2^16 (32768 slots) the build fails exactly as the
    reference's does ("output needs 65536 slots")."""
    rng = np.random.default_rng(seed)
    layers, C, i = [], 3, 0
    for block, (F, n) in enumerate(((64, 2), (128, 2), (256, 3), (512, 3), (512, 3)), start=1):
        for u in range(n):
            i += 1
            layers.append(_conv(f"conv{block}_{u + 1}", F, C, 3, rng, math.sqrt(2.0 / (C * 9)), padding=1,
                                mode="special3x3", bias=False))
            layers.append(Layer("relu", f"relu{block}_{u + 1}", {"degree": 59}))
            C = F
        layers.append(Layer("avg_pool", f"pool{block}", {"kernel": 2, "stride": 2}))
    layers.append(Layer("fc", "fc1", {"outputs": 512}, rng.normal(0, math.sqrt(2.0 / 512), (512, 512)), np.zeros(512)))
    layers.append(Layer("relu", "relu_fc1", {"degree": 59}))
    layers.append(Layer("fc", "fc2", {"outputs": 10}, rng.normal(0, math.sqrt(2.0 / 512), (10, 512)), np.zeros(10)))
    return ModelSpec("vgg16", ring, ring // 2, depth_budget, 3, 32, layers)


def vgg16_paper(seed: int = 5001, ring: int = 65536, depth_budget: int = 11) -> ModelSpec:
    """VGG-16 at the FHEON paper's own widths (the network behind
    its 42.3 GB / 2232 s figure): 3x32x32 input; 3x3 / pad-1 convs 16-16 | 32-32 |
    64-64-64 | 128-128-128 | 128-128-128, 2x2 average pooling after each block,
    then three FC layers.  The table gives FC 1024->1024->1024->10, but after five
    poolings the tensor is 128x1x1, so the first FC takes the 128 flattened
    values: FC 128->1024, 1024->1024, 1024->10.  The first block's 16x32x32 output
    fits one 32768-slot ciphertext.  He-normal weights, bias 0; degree-59
    Chebyshev ReLU after every conv and the two hidden FC layers."""
    rng = np.random.default_rng(seed)
    layers, C = [], 3
    for block, (F, n) in enumerate(((16, 2), (32, 2), (64, 3), (128, 3), (128, 3)), start=1):
        for u in range(n):
            layers.append(_conv(f"conv{block}_{u + 1}", F, C, 3, rng, math.sqrt(2.0 / (C * 9)), padding=1,
                                mode="special3x3", bias=False))
            layers.append(Layer("relu", f"relu{block}_{u + 1}", {"degree": 59, "scale": 8.0}))
            C = F
        layers.append(Layer("avg_pool", f"pool{block}", {"kernel": 2, "stride": 2}))
    n_in = C
    for i, (m, n) in enumerate(((1024, n_in), (1024, 1024), (10, 1024)), start=1):
        layers.append(Layer("fc", f"fc{i}", {"outputs": m}, rng.normal(0, math.sqrt(2.0 / n), (m, n)), np.zeros(m)))
        if i < 3:
            layers.append(Layer("relu", f"relu_fc{i}", {"degree": 59, "scale": 8.0}))
    return ModelSpec("vgg16_paper", ring, ring // 2, depth_budget, 3, 32, layers)


# ----------------------------------------------------------------- build
@dataclass
class Built:
    type: str
    name: str
    src: Optional[Layer]
    in_shape: Tuple
    out_shape: Tuple
    cost: int = 0
    body: List["Built"] = field(default_factory=list)
    downsample: List["Built"] = field(default_factory=list)


def _conv_cfg(L: Layer, C: int) -> fh.ConvConfig:
    p = L.params
    mode = {"generic": fh.ConvMode.generic, "special3x3": fh.ConvMode.special3x3,
            "grouped": fh.ConvMode.grouped}[p.get("mode", "generic")]
    var = fh.StrideVariant.masked if p.get("stride_variant", "extract") == "masked" else fh.StrideVariant.extract
    return fh.ConvConfig(C, p["out_channels"], p["kernel"], p.get("stride", 1), p.get("padding", 0), mode, var)


def _pow2(v):
    return v >= 2 and (v & (v - 1)) == 0


def _cheb_depth(d):
    return 0 if d <= 0 else (1 if d == 1 else int(d - 1).bit_length() + 1)


def _cost(b: Built) -> int:
    """Declared depth costs (layers_conv.cpp:596-628, layers_misc.cpp:297-322)."""
    L, (packed, C, W, n) = b.src, b.in_shape
    if b.type == "conv":
        return fh.conv_depth_cost(_conv_cfg(L, C), W)
    if b.type == "avg_pool":
        k, S = L.params.get("kernel", 2), L.params.get("stride", 2)
        Wo = fh.conv_output_width(W, k, S, 0)
        if S == 1 and Wo == W:
            return 1
        if L.params.get("stride_variant") == "masked" and _pow2(Wo):
            return 1 + (int(Wo - 1).bit_length() + 1 if S >= 2 else 2)
        return 2
    if b.type == "global_avg_pool":
        return 1
    if b.type == "whole_channel_pool":
        return 2
    if b.type == "fc":
        return 2
    if b.type == "relu":
        return (1 if L.params.get("scale", 1.0) > 1.0 else 0) + _cheb_depth(L.params.get("degree", 59))
    if b.type == "bootstrap":
        return 0
    raise fh.ModelError(f"no depth cost for layer type {b.type}", 2)


def _width(L: Layer, W: int, k: int, S: int, P: int) -> int:
    try:
        return fh.conv_output_width(W, k, S, P)
    except fh.Error as e:
        _fail(f"layer '{L.name}': {e}")


def _describe(shape) -> str:
    packed, C, W, n = shape
    return f"{C}x{W}x{W} packed" if packed else f"{n} flat"


def _resolve(layers: List[Layer], shape, slots) -> Tuple[List[Built], Tuple]:
    """resolve_entry (model_spec.cpp:459-716): shape flow and the reference's checks."""
    out = []
    for L in layers:
        packed, C, W, n = shape
        if L.type == "conv":
            if not packed:
                _fail(f"layer '{L.name}': convolution needs a packed tensor input, the flow here is "
                      f"{_describe(shape)}")
            cfg = _conv_cfg(L, C)
            F, k = cfg.out_channels, cfg.kernel
            if F == 0 or k == 0 or cfg.stride == 0:
                _fail(f"layer '{L.name}': out_channels, kernel and stride must be positive")
            mode = L.params.get("mode", "generic")
            if mode == "special3x3":
                if k != 3 or cfg.stride != 1 or cfg.padding != 1:
                    _fail(f"layer '{L.name}': special3x3 mode requires kernel 3, stride 1, padding 1")
                if W < 2:
                    _fail(f"layer '{L.name}': special3x3 mode requires input edge >= 2")
            if mode == "grouped" and F % C != 0:
                _fail(f"layer '{L.name}': grouped convolution requires out_channels ({F}) divisible by the group "
                      f"count ({C})")
            Wo = _width(L, W, k, cfg.stride, cfg.padding)
            Wp = W if mode == "special3x3" else W + 2 * cfg.padding
            if C * Wp * Wp > slots:
                _fail(f"layer '{L.name}': padded input needs {C * Wp * Wp} slots, context provides {slots}")
            new = (True, F, Wo, 0)
            if F * Wo * Wo > slots:
                _fail(f"layer '{L.name}': output needs {F * Wo * Wo} slots, context provides {slots}")
        elif L.type == "avg_pool":
            if not packed:
                _fail(f"layer '{L.name}': pooling needs a packed tensor input")
            k, S = L.params.get("kernel", 2), L.params.get("stride", 2)
            if k == 0 or S == 0:
                _fail(f"layer '{L.name}': kernel and stride must be positive")
            Wo = _width(L, W, k, S, 0)
            if C * Wo * Wo > slots:
                _fail(f"layer '{L.name}': output does not fit in the slot count")
            new = (True, C, Wo, 0)
        elif L.type in ("global_avg_pool", "whole_channel_pool"):
            if not packed:
                _fail(f"layer '{L.name}': pooling needs a packed tensor input")
            if L.type == "whole_channel_pool" and L.params.get("kernel") != W:
                _fail(f"layer '{L.name}': whole-channel pooling requires kernel ({L.params.get('kernel')}) == input "
                      f"edge ({W})")
            new = (False, 0, 0, C)
        elif L.type == "fc":
            have = C * W * W if packed else n
            p = L.params
            if p.get("inputs") and p["inputs"] != have:
                _fail(f"layer '{L.name}': declares {p['inputs']} inputs but receives {have} ({_describe(shape)})")
            if p["outputs"] == 0:
                _fail(f"layer '{L.name}': outputs must be positive")
            if p.get("merge_budget", 1) == 0:
                _fail(f"layer '{L.name}': merge_budget must be >= 1")
            if p["outputs"] > slots or have > slots:
                _fail(f"layer '{L.name}': does not fit in the slot count")
            new = (False, 0, 0, p["outputs"])
        elif L.type == "relu":
            if L.params.get("degree", 59) < 0:
                _fail(f"layer '{L.name}': degree must be >= 0")
            if not L.params.get("scale", 1.0) > 0.0:
                _fail(f"layer '{L.name}': scale must be positive")
            new = shape
        elif L.type == "bootstrap":
            new = shape
        elif L.type == "residual":
            if not packed:
                _fail(f"layer '{L.name}': residual units need packed tensors")
            body, bshape = _resolve(L.body, shape, slots)
            ds, dshape = _resolve(L.downsample, shape, slots) if L.downsample else ([], shape)
            if bshape != dshape or not bshape[0]:
                _fail(f"layer '{L.name}': body produces {_describe(bshape)} but the skip path carries "
                      f"{_describe(dshape)}")
            b = Built("residual", L.name, L, shape, bshape, body=body, downsample=ds)
            out.append(b)
            shape = bshape
            continue
        else:
            _fail(f"unsupported layer type '{L.type}'")
        b = Built(L.type, L.name, L, shape, new)
        b.cost = _cost(b)
        out.append(b)
        shape = new
    return out, shape


def _standard_placement(layers: List[Built], counters: List[int], inserted: List[int]):
    """Bootstrap before every activation past the second, before the second
    pooling layer and before every global reduction (model_spec.cpp:746-776);
    counters run across residual nesting in execution order."""
    i = 0
    while i < len(layers):
        b = layers[i]
        want = False
        if b.type == "relu":
            want = counters[0] >= 2
            counters[0] += 1
        elif b.type == "avg_pool":
            want = counters[1] == 1
            counters[1] += 1
        elif b.type in ("global_avg_pool", "whole_channel_pool"):
            want = True
            counters[1] += 1
        elif b.type == "residual":
            _standard_placement(b.body, counters, inserted)
            i += 1
            continue
        if want and (i == 0 or layers[i - 1].type != "bootstrap"):
            layers.insert(i, Built("bootstrap", f"bootstrap_auto_{inserted[0]}", None, b.in_shape, b.in_shape))
            inserted[0] += 1
            i += 1
        i += 1


def _ledger(layers: List[Built], entry: int, budget: int, inserted: List[int], repair: bool = True) -> int:
    """Level ledger with repair (model_spec.cpp:789-851): a layer that needs
    more levels than remain gets a bootstrap inserted in front of it (policy
    auto) or fails the build (policy explicit)."""
    level = entry
    i = 0
    while i < len(layers):
        b = layers[i]
        if b.type == "bootstrap":
            level = budget
            i += 1
            continue
        need = b.cost
        if b.type == "residual":
            need = b.downsample[0].cost if b.downsample else 0
        if need > level:
            if not repair:
                _fail(f"layer '{b.name}' needs {need} levels but only {level} remain; the explicit bootstrap "
                      f"placement does not hold the depth budget")
            if need > budget:
                raise fh.ModelError(f"layer '{b.name}' needs {need} levels but the depth budget is only {budget}", 2)
            layers.insert(i, Built("bootstrap", f"bootstrap_auto_{inserted[0]}", None, b.in_shape, b.in_shape))
            inserted[0] += 1
            level = budget
            i += 1
        if b.type == "residual":
            d_skip = b.downsample[0].cost if b.downsample else 0
            body_exit = _ledger(b.body, level, budget, inserted, repair)
            ex = min(body_exit, level - d_skip)
            b.cost = level - ex
            level = ex
        else:
            level -= b.cost
        i += 1
    return level


def build(spec: ModelSpec) -> List[Built]:
    """build_model (model_spec.cpp:864-904)."""
    if spec.input_channels == 0 or spec.input_width == 0:
        _fail("model input needs positive channels and width")
    if not spec.layers:
        _fail("model has no layers")
    need = spec.input_channels * spec.input_width * spec.input_width
    if need > spec.slot_count:
        _fail(f"model input needs {need} slots, context provides {spec.slot_count}")
    shape = (True, spec.input_channels, spec.input_width, 0)
    layers, _ = _resolve(spec.layers, shape, spec.slot_count)
    inserted = [0]
    if spec.bootstrap_policy == "auto":
        _standard_placement(layers, [0, 0], inserted)
    _ledger(layers, spec.depth_budget, spec.depth_budget, inserted, spec.bootstrap_policy == "auto")
    return layers


def ends_block(b: Built) -> bool:
    """BuiltLayer::ends_block (model_spec.cpp:521, 555, 577, 708-710): the layer
    shrinks the spatial grid -- a strided conv or pool, a global reduction, or
    a residual unit containing one."""
    L = b.src
    if b.type == "conv":
        return int(L.params.get("stride", 1)) > 1
    if b.type == "avg_pool":
        return int(L.params.get("stride", 2)) > 1
    if b.type in ("global_avg_pool", "whole_channel_pool"):
        return True
    if b.type == "residual":
        return any(ends_block(c) for c in b.body) or (bool(b.downsample) and ends_block(b.downsample[0]))
    return False


def ledger_rows(layers: List[Built], budget: int) -> List[Tuple[str, int, int, bool]]:
    """Top-level (name, level_in, level_out, is_bootstrap) rows the built model
    will record (the reference infer()'s report rows), without running it."""
    rows, level = [], budget
    for b in layers:
        out = budget if b.type == "bootstrap" else level - b.cost
        rows.append((b.name, level, out, b.type == "bootstrap"))
        level = out
    return rows


def count_bootstraps(layers: List[Built]) -> int:
    n = 0
    for b in layers:
        n += b.type == "bootstrap"
        n += count_bootstraps(b.body)
    return n


# ----------------------------------------------------------------- engine
def ckks_config(spec: ModelSpec, bootstrapping: bool, seed: int = 1, schedule: str = "fast",
                security: int = 128, boot_levels: Tuple[int, int] = (0, 0), boot_sparse: int = 3) -> fh.ContextConfig:
    """RNS chain for the spec's ring and depth budget: 55-bit q0, 40-bit
    application primes, 55-bit bootstrapping levels (+16 levels), digits
    balanced by prime bit size, 60-bit special primes (the fewest whose product
    exceeds the widest digit by 2 bits).

    security > 0 (default 128): a uniform ternary secret (bootstrapping through
    the sparse-secret encapsulation, its CoeffsToSlots / EvalMod levels at 60
    bits: the dense secret's rounding noise is ~26x the h = 64 one, and the
    SlotsToCoeffs map amplifies EvalMod noise by sqrt(S) q0 / (2 pi Delta_0);
    the SlotsToCoeffs ramp 60 -> 40 bits runs on "free" plaintext-only levels,
    params.cpp) and the fewest key-switching digits dnum >= 3
    whose chain fits the HE-standard log2(QP) bound for N at `security` bits --
    more digits mean a narrower widest digit, so fewer special primes.  Raises
    ModelError when no dnum fits (e.g. the reference's depth budget 25 with
    bootstrapping at N = 2^16: log2(Q) alone exceeds 1747).
    security = 0: the round-1 chain kept for the reference's presets -- sparse
    h = 64 main secret, dnum 3, allow_insecure (disclosed in host_security).
    boot_sparse: sparse-slot bootstrapping variants over S/2 .. S/2^boot_sparse
    slots (the model's bootstraps carry only the tensor's active slots)."""
    N = spec.ring_dimension
    if spec.slot_count != N // 2:
        raise fh.ShapeError("the engine packs fully: slot_count must be ring_dimension / 2", 2)
    secure = security > 0
    # 128-bit chains: the encapsulation's ephemeral secret at h_b = 32 (sigma(I) = 1.66) with
    # EvalMod range K = 12 (7.2 sigma): a lower-degree cosine, one bootstrapping level less
    boot_hw, boot_kr = (32, 12) if secure else (0, 0)

    def config(K, dnum, L=1):
        return fh.ContextConfig(N, N // 2, spec.depth_budget if not bootstrapping else -1,
                                fh.CryptoMetadata(55, 40, dnum), limbs=L, special_limbs=K, special_bits=60, seed=seed,
                                hamming_weight=0 if (secure or not bootstrapping) else 64, bootstrap=bootstrapping,
                                boot_scale_bits=(60 if secure else 55) if bootstrapping else 0, schedule=schedule,
                                digit_split=1, boot_hamming_weight=boot_hw, boot_k_range=boot_kr,
                                boot_cts_levels=boot_levels[0], boot_stc_levels=boot_levels[1],
                                boot_sparse=boot_sparse if bootstrapping else 0,
                                security=security if secure else 128, allow_insecure=not secure)

    boot_depth = fh.host_bootstrap_depth(config(1, 3)) if bootstrapping else 0
    L = spec.depth_budget + 1 + boot_depth
    _config = config

    def config(K, dnum):  # noqa: F811 -- the chain's limb count fixed from here on
        return _config(K, dnum, L)

    def smallest_k(dnum):
        # digits balanced by bit size over the real Q chain (the special primes are
        # chosen after it, so K does not change it)
        qbits = [math.log2(float(q)) for q in fh.host_primes(config(1, dnum))[0][:L]]
        widest = balanced_widest(qbits, dnum)
        K = max(1, -(-int(widest + 2.0) // 59))
        while K < 16:
            cfg = config(K, dnum)
            pbits = sum(math.log2(float(q)) for q in fh.host_primes(cfg)[0][L:])
            if pbits > widest:
                return cfg
            K += 1
        return None

    if not secure:
        return smallest_k(3)
    last = None
    for dnum in range(3, min(L, 16) + 1):
        cfg = smallest_k(dnum)
        if cfg is None:
            continue
        sec = fh.host_security(cfg)
        last = sec
        if sec["security_bits"] is not None and sec["security_bits"] >= security:
            return cfg
    raise fh.ModelError(f"no {security}-bit chain for depth budget {spec.depth_budget} at N = {N}"
                        + (" with bootstrapping" if bootstrapping else "")
                        + (f": log2(QP) >= {last['log2_qp']} > {last['he_standard_128_bound']}" if last else "")
                        + "; lower the depth budget or pass security=0 (insecure)", 2)


def balanced_widest(bits: List[float], dnum: int, max_size: int = 15) -> float:
    """Widest digit (bits) of the balanced contiguous digit split -- the same
    bisection + greedy packing as params.cpp balanced_digits."""
    def split(cap):
        n, acc, size = 1, 0.0, 0
        for b in bits:
            if b > cap:
                return None
            if size == max_size or acc + b > cap:
                n, acc, size = n + 1, 0.0, 0
            acc += b
            size += 1
        return n if n <= dnum else None

    lo, hi = 0.0, sum(bits)
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if split(mid) is not None:
            hi = mid
        else:
            lo = mid
    return hi


@dataclass
class InferResult:
    logits: np.ndarray
    ledger: List[Tuple[str, int, int, int, bool]]  # name, declared, level_in, level_out, bootstrap
    wall_ms: float
    layer_ms: Dict[str, float]
    stats: Dict[str, int]
    # keyplan (model_run.cpp:148-153): the plan under the requested key mode, the
    # trace replayed against it, and key residency observed on the engine
    plan: Optional[keyplan.BlockPlan] = None
    trace_check: Optional[keyplan.TraceCheck] = None
    key_residency: Optional[Dict[str, int]] = None


class EncryptedModel:
    """A built model bound to an engine context (keys generated on first use)."""

    def __init__(self, spec: ModelSpec, seed: int = 1, schedule: str = "fast", security: int = 128,
                 boot_levels: Tuple[int, int] = (0, 0), boot_sparse: int = 3):
        """security: HE-standard level the chain must meet (ckks_config); 0 runs
        the insecure round-1 chain the reference's presets need (disclosed in
        self.security).  boot_sparse: sparse-slot bootstrapping variants (0 = every
        bootstrap runs the full-slot pipeline)."""
        self.spec = spec
        self.layers = build(spec)
        self.n_boot = count_bootstraps(self.layers)
        self.ctx = fh.SlotContext(ckks_config(spec, self.n_boot > 0, seed, schedule, security, boot_levels,
                                              boot_sparse))
        self.security = self.ctx.security()
        self._layer_keys: Optional[List[keyplan.LayerKeys]] = None
        self.batch_relu = True  # forward_batch: activations of a batch in one polynomial evaluation
        self._pinned_keys = self.ctx.key_count()  # relinearisation / bootstrapping keys made at creation
        if spec.weight_mode == "lazy":
            self.ctx.set_weight_cache(0)
        if self.ctx.depth_budget() != spec.depth_budget:
            raise fh.InternalError("engine depth budget differs from the spec", 3)

    def _run(self, b: Built, v, timings):
        L = b.src
        packed, C, W, n = b.in_shape
        t0 = time.perf_counter()
        if b.type == "conv":
            w = fh.KernelTensor(L.weights, L.bias)
            out = fh.convolution(fh.PackedTensor(v, C, W), _conv_cfg(L, C), w).data
        elif b.type == "avg_pool":
            cfg = fh.PoolConfig(fh.PoolKind.average, L.params.get("kernel", 2), L.params.get("stride", 2),
                                fh.StrideVariant.masked if L.params.get("stride_variant") == "masked"
                                else fh.StrideVariant.extract)
            out = fh.avg_pool(fh.PackedTensor(v, C, W), cfg).data
        elif b.type == "global_avg_pool":
            out = fh.global_avg_pool(fh.PackedTensor(v, C, W))
        elif b.type == "whole_channel_pool":
            out = fh.whole_channel_pool(fh.PackedTensor(v, C, W), L.params.get("kernel", W))
        elif b.type == "fc":
            nin = C * W * W if packed else n
            out = fh.fully_connected(v, fh.FcConfig(nin, L.params["outputs"], L.params.get("merge_budget", 1)),
                                     fh.FcWeights(L.weights, L.bias))
        elif b.type == "relu":
            active = C * W * W if packed else n
            out = fh.secure_relu(v, fh.ReluConfig(L.params.get("scale", 1.0), L.params.get("degree", 59), active))
        elif b.type == "bootstrap":
            # only the tensor's active slots survive (a sparse-slot variant when one fits;
            # a convolution's output is zero past them, so it needs no mask level)
            out = fh.bootstrap(v, C * W * W if packed else n, clean=getattr(v, "_clean", False))
        elif b.type == "residual":
            body = v
            for c in b.body:
                body = self._run(c, body, timings)
            skip = v
            for c in b.downsample:
                skip = self._run(c, skip, timings)
            out = fh.add(body, skip)
            out._clean = getattr(body, "_clean", False) and getattr(skip, "_clean", False)
        else:
            raise fh.ModelError(f"unexecutable layer {b.type}", 2)
        if b.type == "conv":
            # convolutions end in masked placements: slots past F * W_out^2 are zero
            # (layers_conv.cpp:142-177; checked against the reference in test_gpu_layers)
            out._clean = True
        if timings is not None:
            self.ctx.sync()
            timings[b.name] = timings.get(b.name, 0.0) + (time.perf_counter() - t0) * 1e3
        return out

    def _run_batch(self, b: Built, vs: List, timings=None) -> List:
        """One layer on the images of a batch in lockstep (model_run.cpp:100-159 once
        per image): bootstraps run together through bootstrap_many, so each
        bootstrapping key and encoded diagonal is read from HBM once per batch and the
        NTT / basis-conversion launches carry the whole batch; the other layers run
        image by image on the same stream.  Per image the operations are those of
        _run (outputs bit-identical)."""
        packed, C, W, n = b.in_shape
        if b.type == "bootstrap":
            clean = all(getattr(v, "_clean", False) for v in vs)
            return fh.bootstrap_many(vs, C * W * W if packed else n, clean=clean)
        if b.type == "relu" and self.batch_relu:
            L = b.src
            active = C * W * W if packed else n
            return fh.secure_relu_many(vs, fh.ReluConfig(L.params.get("scale", 1.0), L.params.get("degree", 59),
                                                         active))
        if b.type == "residual":
            body = vs
            for c in b.body:
                body = self._run_batch(c, body, timings)
            skip = vs
            for c in b.downsample:
                skip = self._run_batch(c, skip, timings)
            outs = []
            for bd, sk in zip(body, skip):
                o = fh.add(bd, sk)
                o._clean = getattr(bd, "_clean", False) and getattr(sk, "_clean", False)
                outs.append(o)
            return outs
        return [self._run(b, v, timings) for v in vs]

    def forward_batch(self, vs: List[fh.SlotVector]) -> List[fh.SlotVector]:
        """forward() on several encrypted images in lockstep (one stream, one host
        thread): see _run_batch."""
        vs = list(vs)
        for b in self.layers:
            vs = self._run_batch(b, vs)
        return vs

    def infer_batch(self, xs: List[np.ndarray]) -> List[np.ndarray]:
        """Encrypt every image, forward_batch, decrypt: the logits per image."""
        outs = self.forward_batch([self.encrypt_input(x) for x in xs])
        m = self.output_count()
        return [o.slots()[:m].copy() for o in outs]

    def layer_keys(self) -> List[keyplan.LayerKeys]:
        """Per top-level layer, the rotation indices (with use counts) this engine
        issues -- BuiltModel::layer_keys (model_spec.cpp:944-950), derived by one
        recorded probe inference instead of the reference's derive_* algebra (the
        rotation schedule depends on shapes only; under the reference schedule the
        sets equal the reference's).  Cached."""
        if self._layer_keys is None:
            x = np.zeros((self.spec.input_channels, self.spec.input_width, self.spec.input_width))
            rec = self.ctx.attach_recorder()
            try:
                v = fh.SlotVector.encode(self.ctx, x.reshape(-1))
                out = []
                for b in self.layers:
                    rec.clear()
                    v = self._run(b, v, None)
                    ks = keyplan.KeySet()
                    for t in rec.rotation_indices():
                        ks.add(t)
                    out.append(keyplan.LayerKeys(b.name, ks, ends_block(b)))
            finally:
                self.ctx.detach_recorder()
            self._layer_keys = out
        return self._layer_keys

    def memory_model(self) -> keyplan.MemoryModel:
        """MemoryModel::for_context with the engine's true key size; the keys made at
        context creation (relinearisation, conjugation, bootstrapping) are the fixed part."""
        c = self.ctx
        return keyplan.MemoryModel.for_engine(c.N, c.L, c.K, c.dnum, self._pinned_keys)

    def clone(self) -> "EncryptedModel":
        """The same built model on a key-sharing context clone (SlotContext.clone):
        run it from a second host thread to keep two images in flight on the GPU."""
        twin = EncryptedModel.__new__(EncryptedModel)
        twin.__dict__.update(self.__dict__)
        twin.ctx = self.ctx.clone()
        twin._key_store = None
        return twin

    def enable_key_streaming(self):
        """Keyplan block mode WITHOUT regenerating keys on the device: every rotation
        key of the plan is serialized once (packed wire format) into pinned host
        memory, and infer(key_mode="block") then uploads each block's missing keys
        from there on the upload stream (fheon_key_upload_packed_async) -- the
        deployment shape where the server does not hold the secret.  Keys are
        strict while streaming: a key outside the plan is an error, not a silent
        regeneration."""
        import torch
        plan = keyplan.plan_blocks(self.layer_keys())
        store = {}  # by Galois element: rotation steps t and t - S share a key
        for t in plan.union_keys.indices():
            g = self.ctx.galois_element(t)
            if g == 1 or g in store:
                continue
            self.ctx.prefetch_rotation_keys([t])
            buf = torch.empty(self.ctx.key_packed_words(), dtype=torch.uint64, pin_memory=True)
            store[g] = self.ctx.key_download_packed(g, out=buf.numpy())
        self._key_store = store
        self._streamed = set(store)  # Galois elements resident right now

    def output_count(self) -> int:
        packed, C, W, n = self.layers[-1].out_shape
        return C * W * W if packed else n

    def encrypt_input(self, x: np.ndarray) -> fh.SlotVector:
        """SlotVector::encode of the flattened input tensor at the depth budget."""
        x = np.asarray(x, np.float64)
        if x.shape != (self.spec.input_channels, self.spec.input_width, self.spec.input_width):
            raise fh.ShapeError(f"input tensor is {x.shape}, the model expects "
                                f"{(self.spec.input_channels, self.spec.input_width, self.spec.input_width)}", 2)
        return fh.SlotVector.encode(self.ctx, x.reshape(-1))

    def forward(self, v: fh.SlotVector) -> fh.SlotVector:
        """The encrypted forward pass alone: an input ciphertext resident in HBM to
        the logits ciphertext (preload key residency, no host synchronisation
        beyond the engine's own)."""
        for b in self.layers:
            v = self._run(b, v, None)
        return v

    def infer(self, x: np.ndarray, time_layers: bool = False, key_mode: str = "preload",
              verify_keys: bool = False) -> InferResult:
        """Encrypt, run every layer on the GPU, decrypt the logits (model_run.cpp:100-159).

        key_mode (model.hpp:52 KeyMode, model_run.cpp:150): "preload" keeps every
        rotation key resident (generated on first use); "block" makes the keys of
        plan_blocks' block b resident before its first layer and drops, after its
        last layer, those the next block does not use (pinned relinearisation /
        bootstrapping keys stay) -- peak key memory = the largest block instead of
        the union.  verify_keys records the trace with layer markers and replays it
        against the plan (verify_trace)."""
        if key_mode not in ("preload", "block"):
            raise fh.ShapeError(f'key mode must be "preload" or "block", got "{key_mode}"', 2)
        x = np.asarray(x, np.float64)
        if x.shape != (self.spec.input_channels, self.spec.input_width, self.spec.input_width):
            raise fh.ShapeError(f"input tensor is {x.shape}, the model expects "
                                f"{(self.spec.input_channels, self.spec.input_width, self.spec.input_width)}", 2)
        plan = None
        if key_mode == "block" or verify_keys:
            lk = self.layer_keys()
            plan = keyplan.plan_blocks(lk) if key_mode == "block" else keyplan.plan_single_block(lk)
        rec = self.ctx.attach_recorder() if verify_keys else None
        events: List[keyplan.TraceEvent] = []
        store = getattr(self, "_key_store", None) if key_mode == "block" else None
        self.ctx.reset_stats()
        if store is not None:
            self.ctx.set_strict_keys(True)
        peak_key_bytes = 0
        t0 = time.perf_counter()
        v = fh.SlotVector.encode(self.ctx, x.reshape(-1))
        ledger = []
        timings = {} if time_layers else None
        for i, b in enumerate(self.layers):
            if key_mode == "block":
                blk = plan.blocks[plan.block_of_layer(i)]
                if blk.first_layer == i:
                    if i == 0:  # "load block 0": nothing else of the plan stays resident
                        keep = {self.ctx.galois_element(t) for t in blk.keys.indices()}
                        drop = [t for t in plan.union_keys.indices() if self.ctx.galois_element(t) not in keep]
                        self.ctx.drop_rotation_keys(drop)
                        if store is not None:
                            self._streamed -= {self.ctx.galois_element(t) for t in drop}
                    if store is not None:  # stream the block's missing keys from pinned host memory
                        for t in blk.keys.indices():
                            g = self.ctx.galois_element(t)
                            if g in store and g not in self._streamed:
                                self.ctx.key_upload(g, store[g], async_copy=True)
                                self._streamed.add(g)
                    else:
                        self.ctx.prefetch_rotation_keys(blk.keys.indices())
                    peak_key_bytes = max(peak_key_bytes, self.ctx.key_bytes())
            if rec is not None:
                rec.clear()
                events.append(keyplan.TraceEvent("marker", 0, f"layer:{i}:{b.name}"))
            lin = v.level()
            v = self._run(b, v, timings)
            lout = v.level()
            if rec is not None:
                events.extend(keyplan.TraceEvent(e.kind, e.value) for e in rec.snapshot())
            if key_mode == "block":
                bi = plan.block_of_layer(i)
                if plan.blocks[bi].last_layer == i and bi + 1 < len(plan.blocks):
                    nxt = {self.ctx.galois_element(t) for t in plan.blocks[bi + 1].keys.indices()}
                    drop = [t for t in plan.blocks[bi].keys.indices() if self.ctx.galois_element(t) not in nxt]
                    self.ctx.drop_rotation_keys(drop)
                    if store is not None:
                        self._streamed -= {self.ctx.galois_element(t) for t in drop}
            ledger.append((b.name, b.cost, lin, lout, b.type == "bootstrap"))
            if b.type == "bootstrap":
                if lout != self.spec.depth_budget:
                    raise fh.InternalError(f"bootstrap '{b.name}' did not restore the depth budget", 3)
            elif lin - lout != b.cost:
                raise fh.InternalError(f"layer '{b.name}' declared {b.cost} levels but consumed {lin - lout}", 3)
        packed, C, W, n = self.layers[-1].out_shape
        count = C * W * W if packed else n
        logits = v.slots()[:count]
        wall = (time.perf_counter() - t0) * 1e3
        if rec is not None:
            self.ctx.detach_recorder()
        if store is not None:
            self.ctx.wait_transfers()
            self.ctx.set_strict_keys(False)
        up = self.ctx.key_uploads()
        residency = dict(self.ctx.key_events(), peak_key_bytes=max(peak_key_bytes, self.ctx.key_bytes()),
                         resident_key_bytes=self.ctx.key_bytes(), uploaded=up["uploads"], uploaded_bytes=up["bytes"])
        check = keyplan.verify_trace(plan, events) if verify_keys else None
        return InferResult(logits, ledger, wall, timings or {}, self.ctx.stats(), plan, check, residency)


# ----------------------------------------------------------------- calibration
def _forward_float(spec: ModelSpec, x: np.ndarray, maxima: List[float]) -> np.ndarray:
    """True-ReLU float forward (model_run.cpp:161-358 semantics), recording the
    max |pre-activation| of every ReLU site in execution order."""

    def conv(L, t):
        p = L.params
        k, S, P = p["kernel"], p.get("stride", 1), p.get("padding", 0)
        t = np.pad(t, ((0, 0), (P, P), (P, P)))
        C, W, _ = t.shape
        Wo = (W - k) // S + 1
        w = L.weights
        out = np.zeros((w.shape[0], Wo, Wo))
        for i in range(k):
            for j in range(k):
                patch = t[:, i:i + S * (Wo - 1) + 1:S, j:j + S * (Wo - 1) + 1:S]
                out += np.einsum("fc,cab->fab", w[:, :, i, j], patch)
        if L.bias is not None:
            out += L.bias[:, None, None]
        return out

    def run(layers, t):
        for L in layers:
            if L.type == "conv":
                t = conv(L, t)
            elif L.type == "relu":
                maxima.append(float(np.abs(t).max()))
                t = np.maximum(t, 0)
            elif L.type == "avg_pool":
                k, S = L.params.get("kernel", 2), L.params.get("stride", 2)
                C, W, _ = t.shape
                Wo = (W - k) // S + 1
                t = np.stack([[[t[c, a * S:a * S + k, b * S:b * S + k].mean() for b in range(Wo)]
                               for a in range(Wo)] for c in range(C)])
            elif L.type in ("global_avg_pool", "whole_channel_pool"):
                t = t.reshape(t.shape[0], -1).mean(axis=1)
            elif L.type == "fc":
                t = L.weights @ t.reshape(-1) + (L.bias if L.bias is not None else 0)
            elif L.type == "residual":
                body = run(L.body, t)
                skip = run(L.downsample, t) if L.downsample else t
                t = body + skip
        return t

    return run(spec.layers, x)


def calibrate_relu_scales(spec: ModelSpec, batch: List[np.ndarray], safety: float = 1.25) -> ModelSpec:
    """Frozen per-site ReLU scales = max(1, safety * max |pre-activation|) over a
    calibration batch (model_run.cpp:381-403); returns a new spec."""
    per = []
    for x in batch:
        m: List[float] = []
        _forward_float(spec, x, m)
        per.append(m)
    mx = np.max(np.array(per), axis=0)
    spec = copy.deepcopy(spec)
    k = [0]

    def assign(layers):
        for L in layers:
            if L.type == "relu":
                L.params["scale"] = float(max(1.0, safety * mx[k[0]]))
                k[0] += 1
            elif L.type == "residual":
                assign(L.body)

    assign(spec.layers)
    return spec


# ----------------------------------------------------------------- run report
@dataclass
class RunReport:
    """RunReport (model.hpp:211-231): one encrypted inference with its float
    (true-ReLU) reference, per-logit deltas, argmax agreement, ledger, key plan,
    trace check and memory estimate -- plus what the engine adds: the chain's
    security disclosure and its op / launch counters."""
    model_name: str
    kernels: str
    logits: List[float]
    reference_logits: List[float]
    deltas: List[float]
    max_abs_delta: float
    argmax: int
    reference_argmax: int
    argmax_match: bool
    ledger: List[Tuple[str, int, int, int, bool]]
    plan: keyplan.BlockPlan
    trace_check: keyplan.TraceCheck
    memory: keyplan.MemoryEstimate
    rotation_count: int
    wall_ms: float
    notes: List[str]
    security: Dict[str, object]
    engine: Dict[str, object]

    def to_json(self) -> str:
        """The reference's RunReport::to_json layout (model_run.cpp:440-492), same keys
        and nesting, plus "security" and "engine"."""
        j = {"model": self.model_name, "kernels": self.kernels, "logits": list(map(float, self.logits)),
             "reference_logits": list(map(float, self.reference_logits)), "deltas": list(map(float, self.deltas)),
             "max_abs_delta": float(self.max_abs_delta), "argmax": int(self.argmax),
             "reference_argmax": int(self.reference_argmax), "argmax_match": bool(self.argmax_match),
             "rotations": int(self.rotation_count), "wall_ms": float(self.wall_ms),
             "ledger": [{"layer": n, "declared_levels": d, "level_in": li, "level_out": lo, "bootstrap": b}
                        for n, d, li, lo, b in self.ledger],
             "plan": {"blocks": [{"first_layer": b.first_layer, "last_layer": b.last_layer, "keys": b.keys.size()}
                                 for b in self.plan.blocks],
                      "total_keys": self.plan.union_keys.size(), "peak_resident_keys": self.plan.peak_resident_keys,
                      "residency": list(self.plan.residency_events)},
             "trace_check": {"ok": self.trace_check.ok(),
                             "violations": [{"event": v.event_index, "rotation_index": v.rotation_index,
                                             "reason": v.reason} for v in self.trace_check.violations],
                             "unused_keys": list(self.trace_check.unused_keys)},
             "memory": {"total_keys": self.memory.total_keys, "resident_keys": self.memory.resident_keys,
                        "preload_bytes": self.memory.preload_bytes, "peak_bytes": self.memory.peak_bytes,
                        "assumptions": self.memory.assumptions},
             "notes": list(self.notes), "security": self.security, "engine": self.engine}
        return json.dumps(j, indent=2)


def run_with_report(em: EncryptedModel, x: np.ndarray, key_mode: str = "preload") -> RunReport:
    """run_with_report (model_run.cpp:407-437): infer with the trace verified against
    the key plan, the float true-ReLU reference on the same input, and the
    memory estimate under the engine's true key size."""
    r = em.infer(x, key_mode=key_mode, verify_keys=True)
    ref = _forward_float(em.spec, np.asarray(x, np.float64), [])
    n = min(len(r.logits), len(ref))
    deltas = np.abs(np.asarray(r.logits[:n]) - np.asarray(ref[:n]))
    am = int(np.argmax(r.logits)) if len(r.logits) else 0
    ram = int(np.argmax(ref)) if len(ref) else 0
    mem = keyplan.estimate_memory(r.plan, em.memory_model())
    notes = [f"{em.n_boot} bootstraps placed ({em.spec.bootstrap_policy} policy)",
             f"rotation schedule: {em.ctx.schedule()}"]
    engine = {"ring_dimension": em.spec.ring_dimension, "limbs": em.ctx.L, "special_limbs": em.ctx.K,
              "dnum": em.ctx.dnum, "key_mode": key_mode, "key_residency": r.key_residency,
              "ops": {k: int(v) for k, v in r.stats.items()}}
    return RunReport(em.spec.name, "b200 rns-ckks (sm_100a kernels, libfheon_b200.so)", list(r.logits), list(ref),
                     deltas.tolist(), float(deltas.max()) if n else 0.0, am, ram, am == ram,
                     [(a, b, c, d, e) for a, b, c, d, e in r.ledger], r.plan, r.trace_check, mem,
                     r.trace_check.rotations_checked, r.wall_ms, notes, em.security, engine)
