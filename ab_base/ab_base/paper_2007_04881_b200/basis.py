"""Basis specifications (host side) -- mirror of polydg ``basis.py``.

Values and gradients are only ever evaluated on the device
(``csrc/sipg_device.cuh`` ``tabulate_point``); the host keeps the
per-element degree / family / bounding-box metadata and the index-ordering
contract that fixes the matrix block layout (polydg ``basis.py:9-16``):
graded-lexicographic multi-indices, ascending total degree, lexicographic
within a level.
"""

from __future__ import annotations

import itertools
from collections.abc import Sequence
from dataclasses import dataclass
from enum import Enum
from functools import lru_cache
from math import comb

import numpy as np


class Family(Enum):
    P = "P"
    PQ = "PQ"


def family_name(family) -> str:
    """Family of either this package's or polydg's enum (duck-typed)."""
    return getattr(family, "value", family)


@dataclass(frozen=True)
class BasisSpec:
    """Degree, family and box of one element (polydg ``basis.py:36-71``)."""

    degree: int
    family: Family
    box: np.ndarray

    def __post_init__(self):
        box = np.asarray(self.box, dtype=float)
        if box.ndim != 2 or box.shape[0] != 2:
            raise ValueError(f"box must have shape (2, d), got {box.shape}")
        if not np.all(box[1] > box[0]):
            raise ValueError("bounding box must have positive side lengths")
        object.__setattr__(self, "box", box)
        if self.degree < 0:
            raise ValueError("degree must be nonnegative")

    @property
    def dim(self) -> int:
        return self.box.shape[1]

    @property
    def n_funcs(self) -> int:
        return num_basis(self.degree, self.dim, self.family)

    @property
    def total_degree(self) -> int:
        return self.degree if family_name(self.family) == "P" else 2 * self.degree

    def indices(self) -> np.ndarray:
        return multi_indices(self.degree, self.dim, self.family)


def num_basis(p: int, d: int, family=Family.P) -> int:
    if p < 0 or d < 1:
        raise ValueError("need p >= 0 and d >= 1")
    if family_name(family) == "P":
        return comb(p + d, d)
    s = d - 1
    if s < 1:
        raise ValueError("PQ family needs d >= 2")
    return (p + 1) * comb(p + s, s)


@lru_cache(maxsize=None)
def multi_indices(p: int, d: int, family=Family.P) -> np.ndarray:
    """Exponent table (n_funcs, d) in the contract order."""
    levels = []
    for total in range(p + 1):
        levels.extend(a for a in itertools.product(range(total + 1), repeat=d) if sum(a) == total)
    if family_name(family) != "P":
        spatial = []
        for total in range(p + 1):
            spatial.extend(a for a in itertools.product(range(total + 1), repeat=d - 1)
                           if sum(a) == total)
        levels = [(*a, k) for k in range(p + 1) for a in spatial]
    table = np.array(levels, dtype=np.int64).reshape(-1, d)
    table.setflags(write=False)
    return table


class SpecList(Sequence):
    """Array-backed ``list[BasisSpec]``.

    ``build_basis`` returns this so a 4M-element mesh does not materialise
    4M Python objects; indexing yields real ``BasisSpec`` values, so code
    written against polydg's ``list[BasisSpec]`` keeps working.
    """

    def __init__(self, degrees: np.ndarray, boxes: np.ndarray, family=Family.P):
        self.degrees = np.ascontiguousarray(degrees, dtype=np.int64)
        self.boxes = np.ascontiguousarray(boxes, dtype=np.float64)
        self.family = family
        if self.boxes.shape[0] != self.degrees.shape[0]:
            raise ValueError("one box per degree required")

    def __len__(self) -> int:
        return int(self.degrees.shape[0])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        return BasisSpec(int(self.degrees[i]), self.family, self.boxes[i])

    @property
    def dim(self) -> int:
        return int(self.boxes.shape[2])


def build_basis(mesh, degrees, family=Family.P) -> SpecList:
    """Per-element specs on the element bounding boxes (polydg ``basis.py:191-202``)."""
    n = mesh.n_elements
    if np.isscalar(degrees):
        degrees = np.full(n, int(degrees))
    degrees = np.asarray(degrees, dtype=np.int64)
    if degrees.shape != (n,):
        raise ValueError("degrees must be scalar or one per element")
    if np.any(degrees < 0):
        raise ValueError("degree must be nonnegative")
    boxes = np.asarray(mesh.bounding_boxes, dtype=np.float64)
    if not np.all(boxes[:, 1] > boxes[:, 0]):
        raise ValueError("bounding box must have positive side lengths")
    return SpecList(degrees, boxes, family)


def spec_arrays(specs):
    """(degrees int64[nel], boxes f64[nel,2,d], family) of any spec sequence."""
    if isinstance(specs, SpecList):
        return specs.degrees, specs.boxes, specs.family
    specs = list(specs)
    if not specs:
        raise ValueError("empty spec list")
    degrees = np.array([s.degree for s in specs], dtype=np.int64)
    boxes = np.stack([np.asarray(s.box, dtype=np.float64) for s in specs])
    fams = {family_name(s.family) for s in specs}
    if len(fams) != 1:
        raise NotImplementedError("mixed basis families in one assembly")
    return degrees, boxes, specs[0].family
