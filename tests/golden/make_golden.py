"""Generate golden fixtures by running the UNMODIFIED reference implementation.

Run here (the reference is mounted read-only at /root/reference; it does not
exist on the GPU box, so its outputs are committed as fixtures):

    python tests/golden/make_golden.py            # all cases
    python tests/golden/make_golden.py oct cube   # a subset

Each case writes ``<name>.json`` (the network, reference interchange format,
written by the reference's own ``save_network``) and ``<name>.npz``:

* ``seeds``        (S, 3) seed points the reference's trigger produced
* ``keys``         (C, nbytes) uint8 packed canonical states of every visited
                   cell (reference ``marcher.results``), sorted like the
                   reference sorts polygons: by (key bytes, branch)
* ``branch``       (C,) int64, -1 for plain networks
* ``has_face``     (C,) bool, False for empty faces
* ``nverts``       (C,) int64 vertex count per cell (0 for empty)
* ``verts``        (sum nverts, 3) float64, polygon loops in reference order
* ``edge_nrefs``   (sum nverts,) refs per edge; ``edge_refs`` (sum, 2) (kind, index)
* ``report``       JSON string of MarchReport
* ``config``       JSON string of the MarchConfig fields used
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from exactmesh import network as rnet  # noqa: E402  (the reference)
from exactmesh.marching import MarchConfig, march  # noqa: E402
from exactmesh.seeding import sample_seeds  # noqa: E402

from paper_2106_10031_b200 import network as mynet  # noqa: E402
from paper_2106_10031_b200 import synth  # noqa: E402


def make_random_net(depth, width, seed, field_kind="sdf"):
    """Same construction as the reference's tests/conftest.py make_random_net."""
    rng = np.random.default_rng(seed)
    widths = [3] + [width] * depth
    layers = []
    for n_in, n_out in zip(widths[:-1], widths[1:]):
        w = rng.normal(scale=np.sqrt(2.0 / n_in), size=(n_out, n_in))
        b = rng.normal(scale=0.1, size=n_out)
        layers.append(rnet.DenseLayer(w, b))
    head_w = rng.normal(scale=np.sqrt(1.0 / width), size=width)
    net = rnet.NetworkSpec(tuple(layers), head_w, 0.0, field_kind=field_kind)
    probe = rng.uniform(-1.0, 1.0, size=(256, 3))
    med = float(np.median(rnet.forward_many(net, probe)))
    return rnet.NetworkSpec(net.layers, net.head_weight, -med, field_kind=field_kind)


def via_json(my_net, path):
    """Write with our serializer, load with the reference's loader (interchange check)."""
    mynet.save_network(my_net, path)
    return rnet.load_network(path)


def surface_point(net, direction, lo=0.0, hi=1.1):
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    f = lambda t: rnet.forward(net, t * d)  # noqa: E731
    a, b = lo, hi
    fa = f(a)
    for _ in range(200):
        m = 0.5 * (a + b)
        fm = f(m)
        if (fm > 0) == (fa > 0):
            a, fa = m, fm
        else:
            b = m
    return 0.5 * (a + b) * d


def residual_oct():
    oct_net = rnet.octahedron_net(0.5)
    zero6 = rnet.DenseLayer(np.zeros((6, 6)), np.zeros(6))
    return rnet.NetworkSpec((oct_net.layers[0], rnet.ResidualBlock((zero6, zero6))),
                            np.ones(6), -0.5)


def res_linear_random(seed):
    rng = np.random.default_rng(seed)
    l1 = rnet.DenseLayer(rng.normal(scale=0.8, size=(10, 3)), rng.normal(scale=0.1, size=10))
    i1 = rnet.DenseLayer(rng.normal(scale=0.4, size=(8, 10)), rng.normal(scale=0.1, size=8))
    i2 = rnet.DenseLayer(rng.normal(scale=0.4, size=(12, 8)), rng.normal(scale=0.1, size=12))
    blk = rnet.ResidualBlock((i1, i2), rng.normal(scale=0.4, size=(12, 10)),
                             rng.normal(scale=0.1, size=12))
    i3 = rnet.DenseLayer(rng.normal(scale=0.3, size=(12, 12)), rng.normal(scale=0.1, size=12))
    i4 = rnet.DenseLayer(rng.normal(scale=0.3, size=(12, 12)), rng.normal(scale=0.1, size=12))
    idb = rnet.ResidualBlock((i3, i4))
    head = rng.normal(scale=0.3, size=12)
    net = rnet.NetworkSpec((l1, blk, idb), head, 0.0)
    probe = rng.uniform(-1.0, 1.0, size=(256, 3))
    med = float(np.median(rnet.forward_many(net, probe)))
    return rnet.NetworkSpec(net.layers, net.head_weight, -med)


def cases():
    """name -> (builder(path) -> reference net, MarchConfig kwargs, seed_points builder or None)."""
    out = {}
    out["oct"] = (lambda p: via_json(mynet.octahedron_net(0.5), p), dict(seeds=8, rng_seed=3))
    out["cube"] = (lambda p: via_json(mynet.cube_ensemble(0.5), p), dict(seeds=16, rng_seed=5))
    out["oct_occ"] = (lambda p: via_json(mynet.octahedron_net(0.5, field_kind="occupancy"), p),
                      dict(seeds=8, rng_seed=3))
    out["oct_res"] = (lambda p: _save_ref(residual_oct(), p), dict(seeds=8, rng_seed=3))
    out["rand_3x10_s42"] = (lambda p: _save_ref(make_random_net(3, 10, 42), p),
                            dict(seeds=24, rng_seed=7))
    out["rand_4x8_s11"] = (lambda p: _save_ref(make_random_net(4, 8, 11), p),
                           dict(seeds=24, rng_seed=2))
    out["rand_4x12_s13"] = (lambda p: _save_ref(make_random_net(4, 12, 13), p),
                            dict(seeds=32, rng_seed=1))
    out["rand_4x12_s17_cap5"] = (lambda p: _save_ref(make_random_net(4, 12, 17), p),
                                 dict(seeds=8, rng_seed=3, max_cells=5))
    out["rand_6x20_s7"] = (lambda p: _save_ref(make_random_net(6, 20, 7), p),
                           dict(seeds=8, rng_seed=11, max_cells=100000))
    out["res_linear"] = (lambda p: _save_ref(res_linear_random(5), p), dict(seeds=8, rng_seed=4))
    out["deepsdf_small"] = (
        lambda p: via_json(synth.deepsdf_mlp(width=20, depth=5, skip_at=3, bias_std=0.05, seed=3), p),
        dict(seeds=4, rng_seed=0))
    out["imnet_small"] = (
        lambda p: via_json(synth.imnet_ensemble(widths=(12, 12), n_parts=3, seed=1), p),
        dict(seeds=8, rng_seed=0, scheme="dichotomy"))
    # configs[0]: 3-60-60-1 geometric (sphere-SDF) init, single seed point
    out["geo_60x60"] = (lambda p: via_json(synth.geometric_mlp([60, 60], seed=0), p),
                        dict(seeds=1, rng_seed=0))
    # the other two trigger schemes (reference seeding.py:35-77)
    out["rand_3x10_s42_sgd"] = (lambda p: _save_ref(make_random_net(3, 10, 42), p),
                                dict(seeds=6, rng_seed=7, scheme="sgd"))
    out["geo_24x24_sphere"] = (lambda p: via_json(synth.geometric_mlp([24, 24], seed=1), p),
                               dict(seeds=6, rng_seed=2, scheme="sphere_trace"))
    # configs[1] network (3-(90x6)-1) restricted to a sub-box around one surface point
    out["geo_90x6_box"] = (lambda p: via_json(synth.geometric_mlp([90] * 6, seed=0), p),
                           dict(box_around=(0.3, 0.5, 0.8), box_half=0.05))
    return out


def _save_ref(net, path):
    rnet.save_network(net, path)
    return rnet.load_network(path)


def run_case(name, builder, kw):
    jpath = os.path.join(HERE, f"{name}.json")
    net = builder(jpath)
    kw = dict(kw)
    cfg_doc = {}
    if "box_around" in kw:
        p = surface_point(net, kw.pop("box_around"))
        h = kw.pop("box_half")
        bbox = (tuple(p - h), tuple(p + h))
        kw["bbox"] = bbox
        kw["seed_points"] = p.reshape(1, 3)
    cfg = MarchConfig(**kw)
    if cfg.seed_points is None:
        seeds = sample_seeds(net, cfg.seeds, cfg.bbox, scheme=cfg.scheme, rng_seed=cfg.rng_seed)
    else:
        seeds = np.asarray(cfg.seed_points, dtype=np.float64).reshape(-1, 3)
    cfg_doc = {"bbox": [list(cfg.bbox[0]), list(cfg.bbox[1])], "seeds": cfg.seeds,
               "scheme": cfg.scheme, "rng_seed": cfg.rng_seed, "max_cells": cfg.max_cells,
               "explicit_seeds": cfg.seed_points is not None}
    cfg.seed_points = seeds
    t0 = time.perf_counter()
    res = march(net, cfg)
    dt = time.perf_counter() - t0
    # every visited cell, including empty ones, in the reference's sort order
    # (marching.py:346-349 sorts polygons by (key, branch))
    polys = {(p.state.key, p.state.branch): p for p in res.polygons}
    # recover the visited set: polygons + empty states (report counts them)
    visited = list(polys.keys())
    keys, branch, has_face, nverts, verts, enr, erefs = [], [], [], [], [], [], []
    all_states = sorted(set(visited) | set(_empty_states(net, cfg, res)),
                        key=lambda kb: (kb[0], -1 if kb[1] is None else kb[1]))
    for k, b in all_states:
        keys.append(np.frombuffer(k, dtype=np.uint8))
        branch.append(-1 if b is None else b)
        p = polys.get((k, b))
        has_face.append(p is not None)
        if p is None:
            nverts.append(0)
            continue
        nverts.append(p.n_vertices)
        verts.append(p.vertices)
        for refs in p.edge_transitions:
            enr.append(len(refs))
            erefs.extend((r.kind, r.index) for r in refs)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        seeds=seeds,
        keys=np.stack(keys) if keys else np.zeros((0, 1), np.uint8),
        branch=np.asarray(branch, dtype=np.int64),
        has_face=np.asarray(has_face, dtype=bool),
        nverts=np.asarray(nverts, dtype=np.int64),
        verts=np.concatenate(verts) if verts else np.zeros((0, 3)),
        edge_nrefs=np.asarray(enr, dtype=np.int64),
        edge_refs=np.asarray(erefs, dtype=np.int64).reshape(-1, 2),
        report=np.array(res.report.to_json()),
        config=np.array(json.dumps(cfg_doc)),
    )
    print(f"{name}: {len(all_states)} cells ({res.report.faces_emitted} faces, "
          f"{res.report.empty_faces} empty, fallbacks {res.report.pivot_fallbacks}) in {dt:.1f}s")


_EMPTY_CACHE = {}


def _empty_states(net, cfg, res):
    return _EMPTY_CACHE.get(id(res), [])


def _patch_marcher():
    """Record empty-face states: the reference keeps them in _Marcher.results but
    MarchResult only exposes polygons; wrap _Marcher.__init__ to capture the dict."""
    import exactmesh.marching as rm
    orig_init = rm._Marcher.__init__
    holder = {}

    def init(self, *a, **k):
        orig_init(self, *a, **k)
        holder["m"] = self

    rm._Marcher.__init__ = init
    orig_march = rm.march

    def wrapped(net, config=None):
        res = orig_march(net, config)
        m = holder["m"]
        _EMPTY_CACHE[id(res)] = [(s.key, s.branch) for s, p in m.results.items() if p is None]
        return res

    rm.march = wrapped
    globals()["march"] = wrapped


if __name__ == "__main__":
    _patch_marcher()
    want = set(sys.argv[1:])
    for name, (builder, kw) in cases().items():
        if want and name not in want:
            continue
        run_case(name, builder, kw)
