"""paper_2106_10031_b200 -- B200-native analytic marching (exact meshing of ReLU implicit networks).

Drop-in for the reference package's meshing path (exactmesh.march): it marches the
reference's own network objects (or any object with their attributes, see network.py),
reads and writes the same interchange format, and returns the same MarchConfig /
MarchResult / FacePolygon / PolygonMesh shapes, with the marching loop, per-cell affine
maps, face polygons, neighbour generation, the visited set and mesh welding running in
sm_100a CUDA kernels behind a C-ABI library.
"""

from .network import (AffinePlane, DenseLayer, EnsembleSpec, NetworkFormatError, NetworkSpec, RegionMaps,
                      ResidualBlock, StateVector, check_network, cube_ensemble, load_network, network_from_dict,
                      network_to_dict, octahedron_net, region_count_lower_bound, save_network, subnetworks,
                      to_blob)

__all__ = [
    "AffinePlane", "DenseLayer", "EnsembleSpec", "NetworkFormatError", "NetworkSpec", "RegionMaps",
    "ResidualBlock", "StateVector", "check_network", "cube_ensemble", "load_network", "network_from_dict",
    "network_to_dict", "octahedron_net", "region_count_lower_bound", "save_network", "subnetworks", "to_blob",
    "march", "MarchConfig", "MarchResult", "MarchReport", "FacePolygon", "PlaneRef", "Engine",
    "vertex_residuals", "neighbor_state", "forward_many", "forward", "state_at", "state_at_many",
    "affine_maps", "grad_input", "check_unique_planes",
]

__version__ = "0.2.0"

_MARCHING = ("march", "MarchConfig", "MarchResult", "MarchReport", "FacePolygon", "PlaneRef", "vertex_residuals",
             "neighbor_state")
_EVALUATE = ("forward_many", "forward", "state_at", "state_at_many", "affine_maps", "grad_input",
             "check_unique_planes")


def __getattr__(name):
    # the GPU-facing modules import torch; load them on first use
    if name in _MARCHING:
        from . import marching
        return getattr(marching, name)
    if name in _EVALUATE:
        from . import evaluate
        return getattr(evaluate, name)
    if name == "Engine":
        from .engine import Engine
        return Engine
    raise AttributeError(name)
