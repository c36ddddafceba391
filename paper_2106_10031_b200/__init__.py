"""paper_2106_10031_b200 -- B200-native analytic marching (exact meshing of ReLU implicit networks).

Drop-in for the reference package's meshing path (exactmesh.march): same
network model and interchange format, same MarchConfig / MarchResult, with the
marching loop, per-cell affine maps, face polygons, neighbour generation and
the visited set running in sm_100a CUDA kernels behind a C-ABI library.
"""

from .network import (AffinePlane, AnyNetwork, DenseLayer, EnsembleSpec, NetworkFormatError, NetworkSpec,
                      ResidualBlock, StateVector, cube_ensemble, load_network, network_from_dict,
                      octahedron_net, region_count_lower_bound, save_network, subnetworks, to_blob)

__all__ = [
    "AffinePlane", "AnyNetwork", "DenseLayer", "EnsembleSpec", "NetworkFormatError", "NetworkSpec",
    "ResidualBlock", "StateVector", "cube_ensemble", "load_network", "network_from_dict", "octahedron_net",
    "region_count_lower_bound", "save_network", "subnetworks", "to_blob", "march", "MarchConfig",
    "MarchResult", "Engine",
]

__version__ = "0.1.0"


def __getattr__(name):
    # the GPU-facing modules import torch; load them on first use
    if name in ("march", "MarchConfig", "MarchResult", "MarchReport", "FacePolygon", "PlaneRef"):
        from . import marching
        return getattr(marching, name)
    if name == "Engine":
        from .engine import Engine
        return Engine
    raise AttributeError(name)
