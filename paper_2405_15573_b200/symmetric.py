"""Symmetric single-triangle uniform H-matrix (paper Remark 4.5).

A LABELLED VARIANT, not the reference's operator: the reference stores both triangles
(``/root/reference/SPEC.md:8``: "symmetric single-triangle block storage ... both
triangles are stored").  Remark 4.5 (``/root/reference/PAPER.md:488-493``): for a symmetric
(or hermitian) A with I = J and T_I = T_J, use ONE cluster basis X_t per cluster and store
only the admissible blocks below the diagonal; their counterparts above the diagonal are
the transposes.  Here, with V_t = conj(X_t) (symmetric, A^T = A) or V_t = X_t (hermitian,
A^H = A):

  lower admissible block b = (s, t), s after t ......... A|_{s,t} = X_s S_b V_t^H   (stored)
  its mirror (t, s) ...................................... A|_{t,s} = X_t S_b^T V_s^H  (sym)
                                                                    X_t S_b^H V_s^H  (herm)
  lower dense leaf (r, c), r after c .................... D_b (stored), mirror D_b^T / D_b^H
  diagonal dense leaf (r, r) ............................ D_b (stored; symmetric itself)

"s after t" compares the clusters' first indices (tree order); admissible blocks pair
disjoint clusters, so every admissible pair is either lower or upper.  Storage: one basis
set instead of two, half the coupling matrices (each stored as the ell_s x ell_t product),
half the off-diagonal dense leaves.

``expand_uh`` writes the variant out as an ordinary two-triangle UniformHMatrix (of the
mirror types, or of the reference's own types when passed ``uhm_kit.uniform``): that is
how the variant is pinned against the REFERENCE's ``matvec_uh`` (tools/make_golden_sym.py,
tests/test_symmetric.py).  ``symmetrize_uh`` builds the variant from a general operator
(projecting each lower block's column space onto V_t = conj(U_t) / U_t, and symmetrising
the diagonal leaves) -- it changes the operator, by design.

The GPU path (``pack_sym`` + the bulk engine) reads every stored slab ONCE per matvec and
applies it both ways (csrc/uhmv_bulk.cuh: alias pieces + T mode).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .uh_types import ClusterBasis, CoefficientPair, UniformHMatrix

__all__ = [
    "SymmetricUniformHMatrix",
    "lower_blocks",
    "symmetrize_uh",
    "expand_uh",
    "save_sym",
    "load_sym",
    "storage_sym",
]

KINDS = ("symmetric", "hermitian")


def _check_square_tree(bct):
    rt, ct = bct.row_tree, bct.col_tree
    if rt is not ct:
        if len(rt.nodes) != len(ct.nodes) or any(
            a.lo != b.lo or a.hi != b.hi or tuple(a.children) != tuple(b.children) for a, b in zip(rt.nodes, ct.nodes)
        ):
            raise ValueError("a symmetric operator needs T_I = T_J (one cluster tree)")


def lower_blocks(bct):
    """(admissible lower blocks, dense lower-or-diagonal leaves) of a symmetric block tree;
    raises ValueError when the block tree is not symmetric."""
    _check_square_tree(bct)
    rn = bct.row_tree.nodes
    adm = set(bct.admissible_leaves)
    dense = set(bct.inadmissible_leaves)
    low_adm, low_dense = [], []
    for b in bct.admissible_leaves:
        nd = bct.nodes[b]
        mirror = bct.block_of.get((nd.col, nd.row))
        if mirror is None or mirror not in adm:
            raise ValueError(f"block tree not symmetric: admissible block {b} has no admissible mirror")
        if rn[nd.row].lo > rn[nd.col].lo:
            low_adm.append(b)
    for b in bct.inadmissible_leaves:
        nd = bct.nodes[b]
        mirror = bct.block_of.get((nd.col, nd.row))
        if mirror is None or mirror not in dense:
            raise ValueError(f"block tree not symmetric: dense leaf {b} has no dense mirror")
        if rn[nd.row].lo >= rn[nd.col].lo:
            low_dense.append(b)
    return low_adm, low_dense


@dataclass
class SymmetricUniformHMatrix:
    """bct: the (symmetric) block cluster tree; basis: ClusterBasis X_t of every cluster that
    has admissible blocks; coupling: {lower admissible block id: S_b (ell_s x ell_t)};
    dense: {lower or diagonal dense leaf id: D_b}; kind: "symmetric" or "hermitian"."""

    bct: object
    basis: ClusterBasis
    coupling: dict
    dense: dict
    kind: str = "symmetric"

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"kind must be one of {KINDS}")
        low_adm, low_dense = lower_blocks(self.bct)
        if set(self.coupling) != set(low_adm):
            raise ValueError("coupling must hold exactly the lower admissible blocks")
        if set(self.dense) != set(low_dense):
            raise ValueError("dense must hold exactly the lower and diagonal dense leaves")
        dtype = np.dtype(np.float64)
        for m in list(self.basis.matrices.values()) + list(self.coupling.values()) + list(self.dense.values()):
            dtype = np.result_type(dtype, m.dtype)
        self._dtype = dtype

    @property
    def shape(self):
        return self.bct.shape

    def col_basis(self, t):
        """V_t = conj(X_t) (symmetric) or X_t (hermitian)."""
        x = self.basis.matrices[t]
        return np.conj(x) if self.kind == "symmetric" else x

    def mirror(self, m):
        """The transpose used above the diagonal: m^T (symmetric) or m^H (hermitian)."""
        return m.T if self.kind == "symmetric" else np.conj(m).T

    def matvec(self, v, workers: int = 1, adjoint: bool = False):
        from .matvec import matvec_uh_sym

        return matvec_uh_sym(self, v, workers=workers, adjoint=adjoint)


def symmetrize_uh(u, kind: str = "symmetric") -> SymmetricUniformHMatrix:
    """The single-triangle variant of a general UniformHMatrix (reference object or mirror):
    X_t = U_t (row basis); lower block (s, t): S'_b = S_b V_t^H W_t with W_t = conj(U_t)
    (symmetric) or U_t (hermitian), i.e. the block projected onto the new column basis;
    lower dense leaves as stored; diagonal leaves (D + D^T)/2 or (D + D^H)/2."""
    bct = u.bct
    low_adm, low_dense = lower_blocks(bct)
    rb = u.row_basis.matrices
    basis = {}
    for c in set(bct.row_map) | set(bct.col_map):
        if c in rb:
            basis[c] = np.ascontiguousarray(rb[c], dtype=np.complex128)
        else:  # a cluster with column blocks only: its own column basis
            v = u.col_basis.matrices[c]
            basis[c] = np.ascontiguousarray(np.conj(v) if kind == "symmetric" else v, dtype=np.complex128)
    coupling = {}
    for b in low_adm:
        nd = bct.nodes[b]
        pair = u.coeffs[b]
        s_b = pair.s_x @ np.conj(pair.s_y).T
        w_t = np.conj(basis[nd.col]) if kind == "symmetric" else basis[nd.col]
        coupling[b] = np.ascontiguousarray(s_b @ (np.conj(u.col_basis.matrices[nd.col]).T @ w_t), dtype=np.complex128)
    dense = {}
    for b in low_dense:
        nd = bct.nodes[b]
        d = np.asarray(u.dense[b], dtype=np.complex128)
        if nd.row == nd.col:
            d = 0.5 * (d + (d.T if kind == "symmetric" else np.conj(d).T))
        dense[b] = np.ascontiguousarray(d)
    return SymmetricUniformHMatrix(bct, ClusterBasis(basis), coupling, dense, kind)


def expand_uh(us: SymmetricUniformHMatrix, types=None):
    """The variant as an ordinary two-triangle UniformHMatrix (both triangles explicit):
    row basis X, column basis V = conj(X) / X, every admissible block in product form
    (s_x = its coupling, s_y = I), dense leaves mirrored.  ``types``: a module providing
    ClusterBasis / CoefficientPair / UniformHMatrix (e.g. the reference's
    ``uhm_kit.uniform``); default: the mirror types."""
    CB = getattr(types, "ClusterBasis", ClusterBasis)
    CP = getattr(types, "CoefficientPair", CoefficientPair)
    UH = getattr(types, "UniformHMatrix", UniformHMatrix)
    bct = us.bct
    X = us.basis.matrices
    row_basis = {s: X[s] for s in bct.row_map}
    col_basis = {t: np.ascontiguousarray(us.col_basis(t)) for t in bct.col_map}
    coeffs = {}
    for b, s_b in us.coupling.items():
        nd = bct.nodes[b]
        m = bct.block_of[(nd.col, nd.row)]
        coeffs[b] = CP(s_b.copy(), np.eye(s_b.shape[1], dtype=np.complex128))
        sm = np.ascontiguousarray(us.mirror(s_b))
        coeffs[m] = CP(sm, np.eye(sm.shape[1], dtype=np.complex128))
    dense = {}
    for b, d in us.dense.items():
        nd = bct.nodes[b]
        dense[b] = d.copy()
        if nd.row != nd.col:
            dense[bct.block_of[(nd.col, nd.row)]] = np.ascontiguousarray(us.mirror(d))
    dense = {b: dense[b] for b in sorted(dense)}
    return UH(bct, CB(row_basis), CB(col_basis), coeffs, dense)


def storage_sym(us) -> dict:
    """Element counts of the single-triangle storage vs the two-triangle expansion."""
    bct = us.bct
    nodes = bct.row_tree.nodes
    basis = sum(nodes[c].size * m.shape[1] for c, m in us.basis.matrices.items())
    coup = sum(m.size for m in us.coupling.values())
    dense = sum(m.size for m in us.dense.values())
    diag = sum(m.size for b, m in us.dense.items() if bct.nodes[b].row == bct.nodes[b].col)
    full = 2 * basis + 2 * coup + 2 * dense - diag
    return {"basis": basis, "coupling": coup, "dense": dense, "total": basis + coup + dense,
            "two_triangle_total": full, "bytes_estimate": 16 * (basis + coup + dense)}


def save_sym(us, path, **extra) -> None:
    from .uh_io import FORMAT_VERSION, _pack_mats, bct_to_arrays

    arrs = bct_to_arrays(us.bct)
    arrs["format_version"] = np.int64(FORMAT_VERSION)
    arrs["sym_kind"] = np.array(us.kind)
    for key, mats in (("xb", us.basis.matrices), ("sc", us.coupling), ("dn", us.dense)):
        ids = sorted(mats)
        arrs[f"{key}_ids"] = np.asarray(ids, dtype=np.int64)
        arrs[f"{key}_shape"], arrs[f"{key}_data"] = _pack_mats(mats, ids)
    arrs.update({f"x_{k}": np.asarray(v) for k, v in extra.items()})
    np.savez_compressed(path, **arrs)


def load_sym(path):
    """(SymmetricUniformHMatrix, dict of extra arrays)."""
    from .uh_io import _unpack_mats, bct_from_arrays

    with np.load(path) as z:
        d = {k: z[k] for k in z.files}
    bct = bct_from_arrays(d)
    mats = {key: _unpack_mats(d[f"{key}_ids"], d[f"{key}_shape"], d[f"{key}_data"]) for key in ("xb", "sc", "dn")}
    us = SymmetricUniformHMatrix(bct, ClusterBasis(mats["xb"]), mats["sc"], mats["dn"], str(d["sym_kind"]))
    extra = {k[2:]: v for k, v in d.items() if k.startswith("x_")}
    return us, extra
