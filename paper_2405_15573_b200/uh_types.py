"""Host-side mirror of the reference's operator data types (read side only).

The drop-in ``matvec_uh`` accepts the reference's own ``uhm_kit.UniformHMatrix``
(duck-typed) or these mirrors, which carry the same attribute names so the GPU
box -- where the reference package is absent -- can hold operators too.

Mirrored interfaces (reference file:line, relative to /root/reference/pkg/src/uhm_kit):
  Cluster            clustering.py:31-48   (lo, hi, level, bbox, children, size, is_leaf)
  ClusterTree        clustering.py:51-93   (permutation, nodes in DFS preorder, n_min, depth)
  BlockNode          clustering.py:158-170 (row, col, children, admissible)
  BlockClusterTree   clustering.py:173-209 (row_map/col_map/block_of/block_ranges/block_shape)
  ClusterBasis       uniform.py:43-53
  CoefficientPair    uniform.py:56-68      (S_b = s_x @ s_y^H)
  UniformHMatrix     uniform.py:90-117     (_dense_order and _dtype as in __post_init__)
  MatvecStats        hmatrix.py:25-36

Construction (trees, ACA, compression) is NOT mirrored: it stays in the reference.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Cluster",
    "ClusterTree",
    "BlockNode",
    "BlockClusterTree",
    "ClusterBasis",
    "CoefficientPair",
    "UniformHMatrix",
    "MatvecStats",
    "SVDForm",
    "HMatrix",
]


@dataclass
class Cluster:
    index: int
    lo: int
    hi: int
    level: int
    bbox: object = None
    children: tuple = ()

    @property
    def size(self) -> int:
        return self.hi - self.lo

    @property
    def is_leaf(self) -> bool:
        return not self.children


@dataclass
class ClusterTree:
    permutation: np.ndarray
    nodes: list
    n_min: int
    root: int = 0

    @property
    def size(self) -> int:
        return len(self.permutation)

    @property
    def depth(self) -> int:
        return max(c.level for c in self.nodes) + 1

    def leaves(self) -> list:
        return [c for c in self.nodes if c.is_leaf]


@dataclass
class BlockNode:
    index: int
    row: int
    col: int
    children: tuple = ()
    admissible: bool = False

    @property
    def is_leaf(self) -> bool:
        return not self.children


@dataclass
class BlockClusterTree:
    row_tree: ClusterTree
    col_tree: ClusterTree
    params: object
    nodes: list
    admissible_leaves: list
    inadmissible_leaves: list
    row_map: dict
    col_map: dict
    block_of: dict

    @property
    def row_clusters(self) -> list:
        return sorted(self.row_map)

    @property
    def col_clusters(self) -> list:
        return sorted(self.col_map)

    @property
    def shape(self) -> tuple:
        return (self.row_tree.size, self.col_tree.size)

    def block_shape(self, block_id: int) -> tuple:
        b = self.nodes[block_id]
        return (self.row_tree.nodes[b.row].size, self.col_tree.nodes[b.col].size)

    def block_ranges(self, block_id: int) -> tuple:
        b = self.nodes[block_id]
        r = self.row_tree.nodes[b.row]
        c = self.col_tree.nodes[b.col]
        return (r.lo, r.hi, c.lo, c.hi)


@dataclass
class ClusterBasis:
    matrices: dict

    def rank(self, cid: int) -> int:
        return self.matrices[cid].shape[1]

    def ranks(self) -> dict:
        return {cid: m.shape[1] for cid, m in self.matrices.items()}


@dataclass
class CoefficientPair:
    s_x: np.ndarray  # (l_row, k_b)
    s_y: np.ndarray  # (l_col, k_b)

    @property
    def inner_rank(self) -> int:
        return self.s_x.shape[1]

    def product(self) -> np.ndarray:
        return self.s_x @ self.s_y.conj().T


@dataclass
class UniformHMatrix:
    bct: BlockClusterTree
    row_basis: ClusterBasis
    col_basis: ClusterBasis
    coeffs: dict
    dense: dict
    build_stats: object = None

    def __post_init__(self) -> None:
        shape = self.bct.block_shape
        self._dense_order = sorted(self.dense, key=lambda b: -(shape(b)[0] * shape(b)[1]))
        dtype = np.dtype(np.float64)
        for m in self.row_basis.matrices.values():
            dtype = np.result_type(dtype, m.dtype)
        for d in self.dense.values():
            dtype = np.result_type(dtype, d.dtype)
        self._dtype = dtype

    @property
    def shape(self) -> tuple:
        return self.bct.shape

    def matvec(self, v, workers: int = 1, adjoint: bool = False):
        from .matvec import matvec_uh

        return matvec_uh(self, v, workers=workers, adjoint=adjoint)


@dataclass
class MatvecStats:
    leaves_touched: int = 0
    _lock: threading.Lock = field(default_factory=threading.Lock, repr=False, compare=False)

    def count(self, k: int = 1) -> None:
        with self._lock:
            self.leaves_touched += k


@dataclass
class SVDForm:
    """Mirror of lowrank.SVDForm (lowrank.py:51-64): block ~= U diag(sigma) V^H."""

    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray

    @property
    def rank(self) -> int:
        return len(self.sigma)


@dataclass
class HMatrix:
    """Mirror of hmatrix.HMatrix (hmatrix.py:39-69): SVD-form admissible blocks + dense."""

    bct: BlockClusterTree
    admissible: dict
    dense: dict
    tol_used: object = None

    def __post_init__(self) -> None:
        shape = self.bct.block_shape
        self._adm_order = sorted(self.admissible, key=lambda b: -(self.admissible[b].rank * sum(shape(b))))
        self._dense_order = sorted(self.dense, key=lambda b: -(shape(b)[0] * shape(b)[1]))
        dtype = np.dtype(np.float64)
        for f in self.admissible.values():
            dtype = np.result_type(dtype, f.U.dtype)
        for d in self.dense.values():
            dtype = np.result_type(dtype, d.dtype)
        self._dtype = dtype

    @property
    def shape(self) -> tuple:
        return self.bct.shape

    def matvec(self, v, workers: int = 1, adjoint: bool = False):
        from .matvec import matvec_h

        return matvec_h(self, v, workers=workers, adjoint=adjoint)
