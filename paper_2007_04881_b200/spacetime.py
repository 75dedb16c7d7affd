"""Space-time slabs on the B200 engine -- drop-in for polydg ``spacetime.py``.

A slab is one time interval crossed with a spatial polytopic mesh; its
elements are prisms (spatial element x interval) with bounding boxes
(spatial box x interval).  polydg assembles it through the same Approach-2
engine as the spatial problem with a second geometry provider
(``SlabGeometry``, spacetime.py:133-364):

* volume sub-items are sub-prisms (fine spatial simplex x interval) under
  tensor rules (simplex rule x interval rule of the same order,
  quadrature.py:159-178);
* lateral faces (spatial face x interval, normal (n, 0)) carry the interior /
  Dirichlet / Neumann / inflow / outflow machinery;
* bottom facets (the spatial subdivision at t0) are statically inflow: the
  time jump, with the previous slab's trace (or initial data) as boundary
  values; top facets are outflow (no contribution).

Here the whole slab (volume, lateral faces, bottom facet, RHS) is one fused
sm_100a kernel (``csrc/slab_body.cuh``, runtime-specialised with NVRTC per
coefficient set, degree and family), with the index phase and spatial
geometry frames shared with the spatial engine.  Public names mirror polydg:
``TimePartition``, ``SlabMesh``, ``build_slab``, ``assemble_slab``,
``march``, ``save_solution_vector`` / ``load_solution_vector``.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .basis import Family, SpecList, family_name
from .mesh import MeshError


@dataclass
class TimePartition:
    """Strictly increasing time nodes t_0 = 0 < ... < t_N = T (spacetime.py:58-81)."""

    nodes: np.ndarray

    def __post_init__(self):
        self.nodes = np.asarray(self.nodes, dtype=float)
        if self.nodes.ndim != 1 or self.nodes.shape[0] < 2:
            raise ValueError("need at least two time nodes")
        if np.any(np.diff(self.nodes) <= 0):
            raise ValueError("time nodes must be strictly increasing")

    @classmethod
    def uniform(cls, t_final: float, n_steps: int) -> "TimePartition":
        return cls(np.linspace(0.0, t_final, n_steps + 1))

    @property
    def n_steps(self) -> int:
        return self.nodes.shape[0] - 1

    def interval(self, n: int) -> tuple:
        return float(self.nodes[n]), float(self.nodes[n + 1])


@dataclass
class SlabMesh:
    """One space-time slab: spatial mesh x (t0, t1) (spacetime.py:84-104)."""

    spatial: object
    t0: float
    t1: float

    @property
    def tau(self) -> float:
        return self.t1 - self.t0

    @property
    def dim(self) -> int:
        return self.spatial.dim + 1

    @property
    def n_elements(self) -> int:
        return self.spatial.n_elements

    def prism_volume(self, element: int) -> float:
        return float(self.spatial.element_volumes[element] * self.tau)


def build_slab(spatial_mesh, interval, degrees, family=Family.PQ):
    """Slab mesh plus per-prism basis specs on (spatial box) x interval
    (spacetime.py:107-128)."""
    t0, t1 = float(interval[0]), float(interval[1])
    if not t1 > t0:
        raise ValueError("slab interval must have positive length")
    slab = SlabMesh(spatial_mesh, t0, t1)
    n = spatial_mesh.n_elements
    if np.isscalar(degrees):
        degrees = np.full(n, int(degrees))
    degrees = np.asarray(degrees, dtype=np.int64)
    if degrees.shape != (n,):
        raise ValueError("degrees must be scalar or one per element")
    sbox = np.asarray(spatial_mesh.bounding_boxes, dtype=np.float64)
    boxes = np.empty((n, 2, slab.dim))
    boxes[:, :, :-1] = sbox
    boxes[:, 0, -1], boxes[:, 1, -1] = t0, t1
    return slab, SpecList(degrees, boxes, family)


# -- binary solution dumps (spacetime.py:624-645) --------------------------------

def save_solution_vector(path, vec) -> None:
    """Little-endian binary dump: uint64 length header, then float64 data."""
    vec = np.asarray(vec, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", vec.shape[0]))
        fh.write(vec.tobytes())


def load_solution_vector(path) -> np.ndarray:
    with open(path, "rb") as fh:
        (n,) = struct.unpack("<Q", fh.read(8))
        data = np.frombuffer(fh.read(8 * n), dtype="<f8")
    if data.shape[0] != n:
        raise MeshError(f"{path}: truncated solution vector")
    return data.astype(float)
