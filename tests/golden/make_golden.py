"""Generates the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libslotcnn_ref.so, compiled from /root/reference/proj)
on seeded inputs, plus the reference's own frozen ReLU bound fixture
(proj/tests/data/relu_epsilon59.json) and its model specs (proj/models/*.json).  Run here (container) where
/root/reference exists:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref as sref  # noqa: E402


def events_array(ev):
    kinds = {"rotation": 0, "mult_plain": 1, "mult_cipher": 2, "bootstrap": 3}
    return np.array([(kinds[k], v) for k, v in ev], dtype=np.int64).reshape(-1, 2)


def main():
    # config 1 conv layer (BASELINE configs[0])
    r = sref.Ref(16384, 8192, 10)
    x = np.random.default_rng(1001).uniform(0, 1, (1, 28, 28))
    w = np.random.default_rng(1002).normal(0, 0.1, (6, 1, 5, 5))
    res = r.convolution(x, 10, 1, 28, 6, 5, 1, 0, 0, 0, w, None)
    np.savez_compressed(os.path.join(HERE, "conv_config1.npz"), x=x, w=w, out=res.slots[: 6 * 24 * 24],
                        level=res.level, events=events_array(res.events))
    # small-ring layer cases (ring 4096, 2048 slots, depth 13)
    r = sref.Ref(4096, 2048, 13)
    rng = np.random.default_rng(77)
    x = rng.uniform(-1, 1, (3, 8, 8))
    w = rng.uniform(-1, 1, (4, 3, 3, 3))
    b = rng.uniform(-1, 1, 4)
    res = r.convolution(x, 13, 3, 8, 4, 3, 1, 1, 1, 0, w, b)
    np.savez_compressed(os.path.join(HERE, "special3x3_small.npz"), x=x, w=w, b=b, out=res.slots, level=res.level,
                        events=events_array(res.events))
    res = r.pool(x, 13, 3, 8, 0, 2, 2, 1)
    np.savez_compressed(os.path.join(HERE, "avgpool_masked_small.npz"), x=x, out=res.slots, level=res.level,
                        events=events_array(res.events))
    fw = rng.uniform(-1, 1, (5, 192))
    fb = rng.uniform(-1, 1, 5)
    res = r.fully_connected(x.reshape(-1), 13, 192, 5, 2, fw, fb)
    np.savez_compressed(os.path.join(HERE, "fc_small.npz"), x=x.reshape(-1), w=fw, b=fb, out=res.slots,
                        level=res.level, events=events_array(res.events))
    xr = rng.uniform(-8, 8, 40)
    res = r.secure_relu(xr, 13, 8.0, 59, 40)
    np.savez_compressed(os.path.join(HERE, "relu59_beta8_small.npz"), x=xr, out=res.slots, level=res.level,
                        events=events_array(res.events), coeffs=sref.cheb_relu_coefficients(8.0, 59))
    # the reference's frozen ReLU-approximation bound (proj/tests/data/relu_epsilon59.json)
    src = "/root/reference/proj/tests/data/relu_epsilon59.json"
    d = json.load(open(src))
    json.dump({k: d[k] for k in ("degree", "grid_points", "deadzone", "epsilon_59", "sup_norm")},
              open(os.path.join(HERE, "relu_epsilon59.json"), "w"), indent=1)
    # the reference's own model specs (models/lenet5.json, models/resnet20.json): the
    # architecture descriptions the model runtime must drive; their CSV weights are not
    # shipped, tests/model_files.py materialises seeded ones next to a copy
    specs = {m: json.load(open(f"/root/reference/proj/models/{m}.json")) for m in ("lenet5", "resnet20")}
    with open(os.path.join(HERE, "ref_model_specs.json"), "w") as f:  # one compact line per model
        f.write("{\n" + ",\n".join(f"{json.dumps(m)}: {json.dumps(d, separators=(',', ':'))}"
                                    for m, d in specs.items()) + "\n}\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
