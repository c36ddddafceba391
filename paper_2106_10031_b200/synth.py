"""Synthetic ReLU implicit networks for the BASELINE.json configurations.

There is no network access for checkpoints, so every benchmark network is a
seeded random initialisation of the named architecture:

* ``geometric_mlp`` -- plain ReLU MLP with the geometric (sphere-SDF)
  initialisation of Atzmon & Lipman (SAL, 2020): hidden weights
  N(0, sqrt(2)/sqrt(n_out)), hidden biases 0, head weights
  N(sqrt(pi)/sqrt(n_L), 1e-6), head bias -r.  At init the field is close to
  |x| - r, so the zero set is a sphere-like closed surface of radius ~r.
  configs[0] (3-60-60-1) and configs[1] (3-(90x6)-1).
* ``deepsdf_mlp`` -- DeepSDF-style 3-(512x8)-1: the input x re-enters at
  hidden layer ``skip_at`` (DeepSDF's ``latent_in``).  In the reference's
  layer vocabulary that is a ``residual_linear`` block whose inner stack is
  the first ``skip_at`` layers and whose shortcut V acts on the block input x
  (W_4 [h_3; x] = W_4 h_3 + V x).  configs[2].
* ``imnet_ensemble`` -- IM-NET-style occupancy MLPs merged by a max-pool
  layer (reference EnsembleSpec, paper §5.2).  configs[3].
* ``latent_batch`` -- DeepSDF decoders conditioned on a per-shape 256-d code
  z (input z ⊕ x): with z fixed the code folds into the first-layer and skip
  biases, giving one plain network per shape.  configs[4].
"""

from __future__ import annotations

import numpy as np

from .network import DenseLayer, EnsembleSpec, NetworkSpec, ResidualBlock


def _geo_hidden(rng, n_in, n_out):
    return rng.normal(0.0, np.sqrt(2.0) / np.sqrt(n_out), size=(n_out, n_in))


def _geo_head(rng, n_last):
    return rng.normal(np.sqrt(np.pi) / np.sqrt(n_last), 1e-6, size=n_last)


def geometric_mlp(widths, radius: float = 0.5, seed: int = 0, bias_std: float = 0.0,
                  field_kind: str = "sdf") -> NetworkSpec:
    """SAL geometric init; ``bias_std > 0`` adds N(0, bias_std) hidden biases."""
    rng = np.random.default_rng(seed)
    dims = [3] + list(widths)
    layers = []
    for n_in, n_out in zip(dims[:-1], dims[1:]):
        w = _geo_hidden(rng, n_in, n_out)
        b = rng.normal(0.0, bias_std, size=n_out) if bias_std > 0 else np.zeros(n_out)
        layers.append(DenseLayer(w, b))
    return NetworkSpec(tuple(layers), _geo_head(rng, dims[-1]), -radius, field_kind=field_kind)


def deepsdf_mlp(width: int = 512, depth: int = 8, skip_at: int = 4, radius: float = 0.5,
                seed: int = 0, bias_std: float = 0.0, latent_dim: int = 0,
                latent: np.ndarray | None = None) -> NetworkSpec:
    """DeepSDF decoder with x (and the latent code) re-entering at hidden layer ``skip_at``."""
    return _deepsdf_assemble(_deepsdf_parts(width, depth, skip_at, radius, seed, bias_std, latent_dim), latent)


def _deepsdf_parts(width, depth, skip_at, radius, seed, bias_std, latent_dim):
    """The decoder's arrays (drawn once): the code only enters the first-layer and skip biases."""
    if not 1 <= skip_at < depth:
        raise ValueError("skip_at must be in [1, depth)")
    rng = np.random.default_rng(seed)
    in_dim = 3 + latent_dim
    inner = []
    n_in = in_dim
    for k in range(skip_at):
        w = _geo_hidden(rng, n_in, width)
        b = rng.normal(0.0, bias_std, size=width) if bias_std > 0 else np.zeros(width)
        inner.append((w, b))
        n_in = width
    v_full = _geo_hidden(rng, in_dim, width) / np.sqrt(2.0)
    later = []
    for _ in range(depth - skip_at):
        b = rng.normal(0.0, bias_std, size=width) if bias_std > 0 else np.zeros(width)
        later.append(DenseLayer(_geo_hidden(rng, width, width), b))
    w0 = inner[0][0]
    return {"latent_dim": latent_dim, "inner": inner, "w0x": w0[:, :3] if latent_dim else w0, "v_full": v_full,
            "vx": v_full[:, :3], "later": tuple(later), "head": _geo_head(rng, width), "radius": radius}


def _deepsdf_assemble(parts, latent):
    latent_dim = parts["latent_dim"]
    z = np.zeros(latent_dim) if latent is None else np.asarray(latent, dtype=np.float64)
    inner = []
    for k, (w, b) in enumerate(parts["inner"]):
        if k == 0 and latent_dim:
            # x-part keeps its columns (one shared array); the code part folds into the bias
            inner.append(DenseLayer(parts["w0x"], b + w[:, 3:] @ z))
        else:
            inner.append(DenseLayer(w, b))
    v_full = parts["v_full"]
    vb = v_full[:, 3:] @ z if latent_dim else np.zeros(v_full.shape[0])
    block = ResidualBlock(tuple(inner), parts["vx"], vb)
    return NetworkSpec((block,) + parts["later"], parts["head"], -parts["radius"])


def imnet_ensemble(widths=(64, 64, 64), n_parts: int = 4, seed: int = 0,
                   field_kind: str = "occupancy", spread: float = 0.35,
                   radius: float = 0.3) -> EnsembleSpec:
    """Max-pool union of ``n_parts`` geometric MLPs centred at random points.

    Each part's occupancy logit is -(|x - c_i| - r) shape-wise (positive
    inside), so the union max_i is the occupancy of the union of parts.
    """
    rng = np.random.default_rng(seed)
    subs = []
    for _ in range(n_parts):
        centre = rng.uniform(-spread, spread, size=3)
        dims = [3] + list(widths)
        layers = []
        for li, (n_in, n_out) in enumerate(zip(dims[:-1], dims[1:])):
            w = _geo_hidden(rng, n_in, n_out)
            b = -w @ centre if li == 0 else np.zeros(n_out)
            layers.append(DenseLayer(w, b))
        head = _geo_head(rng, dims[-1])
        # occupancy logit: positive inside (negated SDF), scaled like a logit
        subs.append(NetworkSpec(tuple(layers), -10.0 * head, 10.0 * radius, field_kind=field_kind))
    return EnsembleSpec(tuple(subs))


def latent_batch(n_shapes: int = 64, latent_dim: int = 256, width: int = 512, depth: int = 8,
                 skip_at: int = 4, seed: int = 0, code_std: float = 0.01):
    """One shared DeepSDF decoder, ``n_shapes`` codes z_i ~ N(0, code_std): list of networks (the
    decoder's weight arrays are shared by every network; only the code-folded biases differ)."""
    rng = np.random.default_rng([seed, 1])
    codes = rng.normal(0.0, code_std, size=(n_shapes, latent_dim))
    parts = _deepsdf_parts(width, depth, skip_at, 0.5, seed, 0.0, latent_dim)
    return [_deepsdf_assemble(parts, z) for z in codes], codes


