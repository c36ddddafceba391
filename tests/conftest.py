import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built extension")
    config.addinivalue_line("markers", "slow: long-running case")


def golden_cases():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and not f.startswith("weld_"))


def load_golden(name):
    import json
    from paper_2106_10031_b200.network import load_network
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    g["config"] = json.loads(str(g["config"]))
    g["report"] = json.loads(str(g["report"]))
    g["net"] = load_network(os.path.join(GOLDEN, name + ".json"))
    return g


def make_random_net(depth, width, seed, field_kind="sdf"):
    """Same construction as the reference's tests/conftest.py:7-22 (random He-init MLP)."""
    from paper_2106_10031_b200.network import DenseLayer, NetworkSpec
    import oracle
    rng = np.random.default_rng(seed)
    widths = [3] + [width] * depth
    layers = []
    for n_in, n_out in zip(widths[:-1], widths[1:]):
        w = rng.normal(scale=np.sqrt(2.0 / n_in), size=(n_out, n_in))
        b = rng.normal(scale=0.1, size=n_out)
        layers.append(DenseLayer(w, b))
    head_w = rng.normal(scale=np.sqrt(1.0 / width), size=width)
    net = NetworkSpec(tuple(layers), head_w, 0.0, field_kind=field_kind)
    probe = rng.uniform(-1.0, 1.0, size=(256, 3))
    med = float(np.median(oracle.OracleNet(net).forward_many(probe)))
    return NetworkSpec(net.layers, net.head_weight, -med, field_kind=field_kind)
