"""Materialises a reference model spec (tests/golden/ref_model_specs.json) with
seeded CSV weights for every file it references: the reference ships the
architectures but not the weights (models/README.md)."""
import json
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SPECS = os.path.join(HERE, "golden", "ref_model_specs.json")  # tests/golden/make_golden.py


def _write(path, values):
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savetxt(path, np.asarray(values).reshape(1, -1), delimiter=",", fmt="%.17g")


def materialize(name: str, out_dir: str, seed: int = 1, context=None) -> str:
    """Write the reference's <name> spec (tests/golden/ref_model_specs.json) into
    out_dir (optionally with an inline context replacing the preset) and seeded
    He-normal weights for every CSV it names."""
    spec = json.load(open(REF_SPECS))[name]
    if context is not None:
        spec["context"] = context
    rng = np.random.default_rng(seed)

    def walk(layers, C, W, n, packed):
        for L in layers:
            t = L["type"]
            if t == "conv":
                F, k = L["out_channels"], L["kernel"]
                S, P = L.get("stride", 1), L.get("padding", 0)
                wc = 1 if L.get("mode") == "grouped" else C
                if "weights" in L:
                    _write(os.path.join(out_dir, L["weights"]), rng.normal(0, math.sqrt(2.0 / (wc * k * k)),
                                                                           F * wc * k * k))
                if "bias" in L:
                    _write(os.path.join(out_dir, L["bias"]), rng.normal(0, 0.05, F))
                C, W, packed = F, (W + 2 * P - k) // S + 1, True
            elif t == "batchnorm":
                for key, gen in (("gamma", lambda: rng.uniform(0.8, 1.2, C)), ("beta", lambda: rng.normal(0, 0.05, C)),
                                 ("mean", lambda: rng.normal(0, 0.05, C)), ("var", lambda: rng.uniform(0.8, 1.2, C))):
                    if isinstance(L.get(key), str):
                        _write(os.path.join(out_dir, L[key]), gen())
            elif t == "avg_pool":
                k, S = L.get("kernel", 2), L.get("stride", 2)
                W = (W - k) // S + 1
            elif t in ("global_avg_pool", "whole_channel_pool"):
                n, packed = C, False
            elif t == "fc":
                have = C * W * W if packed else n
                m = L["outputs"]
                if "weights" in L:
                    _write(os.path.join(out_dir, L["weights"]), rng.normal(0, math.sqrt(2.0 / have), m * have))
                if "bias" in L:
                    _write(os.path.join(out_dir, L["bias"]), rng.normal(0, 0.05, m))
                n, packed = m, False
            elif t == "residual":
                C2, W2, n2, p2 = walk(L["layers"], C, W, n, packed)
                if "downsample" in L:
                    walk([L["downsample"]], C, W, n, packed)
                C, W, n, packed = C2, W2, n2, p2
        return C, W, n, packed

    walk(spec["layers"], spec["input"]["channels"], spec["input"]["width"], 0, True)
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, f"{name}.json")
    with open(path, "w") as f:
        json.dump(spec, f, indent=1)
    return path


__all__ = ["materialize", "REF_SPECS"]
