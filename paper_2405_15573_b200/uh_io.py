"""Versioned on-disk format for cluster trees, block trees and uniform H-matrices.

SURVEY.md §8f(3): a ``.npz`` holding the index structure and the operator values so
operators built once by the reference (construction takes minutes to hours) can be
reloaded -- on the GPU box too, where the reference package is absent -- into the
mirror types of :mod:`uh_types`.  Works on the reference's own objects (duck-typed
read of ``clustering.py:31-209`` / ``uniform.py:43-117``) and on the mirrors.

Layout (all integer arrays int64):
  tree  {pfx}_lo, _hi, _level, _child_ptr/_child (CSR), _bbox (n,2,3) or absent, _perm
  bct   blk_row, blk_col, blk_adm, blk_child_ptr/blk_child (CSR), same_tree
  uh    rb_ids/rb_rank/rb_data (row bases, row-major |s| x l_s each, concatenated),
        cb_* (column bases), cf_ids/cf_k/sx_data/sy_data (factorized coefficients),
        dn_ids/dn_data (dense leaves, row-major)
"""

from __future__ import annotations

import numpy as np

from .uh_types import (
    BlockClusterTree,
    BlockNode,
    Cluster,
    ClusterBasis,
    ClusterTree,
    CoefficientPair,
    HMatrix,
    SVDForm,
    UniformHMatrix,
)

FORMAT_VERSION = 1

__all__ = [
    "tree_to_arrays",
    "tree_from_arrays",
    "bct_to_arrays",
    "bct_from_arrays",
    "uh_to_arrays",
    "uh_from_arrays",
    "save_uh",
    "load_uh",
    "save_bct",
    "load_bct",
    "save_h",
    "load_h",
]


class _Box:
    """Minimal AABB mirror (geometry.py:59-70) so ``aabb_dist`` style code works."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo, hi):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)


def _csr(children):
    ptr = np.zeros(len(children) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(c) for c in children])
    flat = np.fromiter((x for c in children for x in c), dtype=np.int64, count=int(ptr[-1]))
    return ptr, flat


def tree_to_arrays(tree, pfx: str) -> dict:
    nodes = tree.nodes
    out = {
        f"{pfx}_lo": np.array([c.lo for c in nodes], dtype=np.int64),
        f"{pfx}_hi": np.array([c.hi for c in nodes], dtype=np.int64),
        f"{pfx}_level": np.array([c.level for c in nodes], dtype=np.int64),
        f"{pfx}_perm": np.asarray(tree.permutation, dtype=np.int64),
        f"{pfx}_nmin": np.int64(tree.n_min),
        f"{pfx}_root": np.int64(getattr(tree, "root", 0)),
    }
    ptr, flat = _csr([tuple(c.children) for c in nodes])
    out[f"{pfx}_child_ptr"] = ptr
    out[f"{pfx}_child"] = flat
    if all(getattr(c, "bbox", None) is not None for c in nodes):
        out[f"{pfx}_bbox"] = np.array([[c.bbox.lo, c.bbox.hi] for c in nodes], dtype=np.float64)
    return out


def tree_from_arrays(d, pfx: str) -> ClusterTree:
    lo, hi, lev = d[f"{pfx}_lo"], d[f"{pfx}_hi"], d[f"{pfx}_level"]
    ptr, flat = d[f"{pfx}_child_ptr"], d[f"{pfx}_child"]
    bb = d[f"{pfx}_bbox"] if f"{pfx}_bbox" in d else None
    nodes = []
    for i in range(len(lo)):
        ch = tuple(int(x) for x in flat[ptr[i] : ptr[i + 1]])
        box = _Box(bb[i, 0], bb[i, 1]) if bb is not None else None
        nodes.append(Cluster(i, int(lo[i]), int(hi[i]), int(lev[i]), box, ch))
    root = int(d[f"{pfx}_root"])
    perm = np.asarray(d[f"{pfx}_perm"])
    if perm.size == 0:  # fixtures may drop the permutation (pinned by a sha256 instead)
        perm = np.arange(int(hi[root]) - int(lo[root]), dtype=np.int64)
    return ClusterTree(perm, nodes, int(d[f"{pfx}_nmin"]), root)


def bct_to_arrays(bct) -> dict:
    same = bct.row_tree is bct.col_tree
    out = tree_to_arrays(bct.row_tree, "rt")
    if not same:
        out.update(tree_to_arrays(bct.col_tree, "ct"))
    nodes = bct.nodes
    out["same_tree"] = np.int64(same)
    out["blk_row"] = np.array([b.row for b in nodes], dtype=np.int64)
    out["blk_col"] = np.array([b.col for b in nodes], dtype=np.int64)
    out["blk_adm"] = np.array([bool(b.admissible) and not b.children for b in nodes], dtype=np.int8)
    ptr, flat = _csr([tuple(b.children) for b in nodes])
    out["blk_child_ptr"] = ptr
    out["blk_child"] = flat
    # the leaf lists as stored (preorder in the reference, clustering.py:227-245)
    out["adm_leaves"] = np.asarray(bct.admissible_leaves, dtype=np.int64)
    out["dense_leaves"] = np.asarray(bct.inadmissible_leaves, dtype=np.int64)
    params = getattr(bct, "params", None)
    if params is not None and hasattr(params, "eta"):
        out["adm_eta"] = np.float64(params.eta)
        out["adm_weak"] = np.int64(params.criterion == "weak")
    return out


class _Params:
    def __init__(self, eta, criterion):
        self.eta = eta
        self.criterion = criterion


def bct_from_arrays(d) -> BlockClusterTree:
    rt = tree_from_arrays(d, "rt")
    ct = rt if int(d["same_tree"]) else tree_from_arrays(d, "ct")
    rows, cols, adm = d["blk_row"], d["blk_col"], d["blk_adm"]
    ptr, flat = d["blk_child_ptr"], d["blk_child"]
    nodes = []
    block_of = {}
    for i in range(len(rows)):
        ch = tuple(int(x) for x in flat[ptr[i] : ptr[i + 1]])
        r, c = int(rows[i]), int(cols[i])
        nodes.append(BlockNode(i, r, c, ch, bool(adm[i])))
        block_of[(r, c)] = i
    adm_leaves = [int(x) for x in d["adm_leaves"]]
    dense_leaves = [int(x) for x in d["dense_leaves"]]
    row_map: dict = {}
    col_map: dict = {}
    for b in adm_leaves:
        r, c = nodes[b].row, nodes[b].col
        row_map.setdefault(r, []).append(c)
        col_map.setdefault(c, []).append(r)
    params = None
    if "adm_eta" in d:
        params = _Params(float(d["adm_eta"]), "weak" if int(d["adm_weak"]) else "strong")
    return BlockClusterTree(rt, ct, params, nodes, adm_leaves, dense_leaves, row_map, col_map, block_of)


def _pack_mats(mats, ids):
    dtype = np.result_type(np.float64, *[mats[i].dtype for i in ids]) if ids else np.dtype(np.float64)
    shapes = np.array([mats[i].shape for i in ids], dtype=np.int64).reshape(-1, 2)
    data = (
        np.concatenate([np.ascontiguousarray(mats[i], dtype=dtype).ravel() for i in ids])
        if ids
        else np.zeros(0, dtype=dtype)
    )
    return shapes, data


def _unpack_mats(ids, shapes, data):
    out = {}
    off = 0
    for i, (r, c) in zip(ids, shapes):
        n = int(r) * int(c)
        out[int(i)] = data[off : off + n].reshape(int(r), int(c)).copy()
        off += n
    return out


def uh_to_arrays(u) -> dict:
    out = bct_to_arrays(u.bct)
    out["format_version"] = np.int64(FORMAT_VERSION)
    for key, basis in (("rb", u.row_basis), ("cb", u.col_basis)):
        ids = sorted(basis.matrices)
        shapes, data = _pack_mats(basis.matrices, ids)
        out[f"{key}_ids"] = np.asarray(ids, dtype=np.int64)
        out[f"{key}_shape"] = shapes
        out[f"{key}_data"] = data
    cids = sorted(u.coeffs)
    sx = {b: u.coeffs[b].s_x for b in cids}
    sy = {b: u.coeffs[b].s_y for b in cids}
    out["cf_ids"] = np.asarray(cids, dtype=np.int64)
    out["sx_shape"], out["sx_data"] = _pack_mats(sx, cids)
    out["sy_shape"], out["sy_data"] = _pack_mats(sy, cids)
    dids = sorted(u.dense)
    out["dn_ids"] = np.asarray(dids, dtype=np.int64)
    out["dn_shape"], out["dn_data"] = _pack_mats(u.dense, dids)
    out["dense_order"] = np.asarray(getattr(u, "_dense_order", dids), dtype=np.int64)
    return out


def uh_from_arrays(d) -> UniformHMatrix:
    bct = bct_from_arrays(d)
    rb = _unpack_mats(d["rb_ids"], d["rb_shape"], d["rb_data"])
    cb = _unpack_mats(d["cb_ids"], d["cb_shape"], d["cb_data"])
    sx = _unpack_mats(d["cf_ids"], d["sx_shape"], d["sx_data"])
    sy = _unpack_mats(d["cf_ids"], d["sy_shape"], d["sy_data"])
    # insertion order of the dense dict follows the stored order so _dense_order ties match
    dn_all = _unpack_mats(d["dn_ids"], d["dn_shape"], d["dn_data"])
    order = [int(b) for b in d["dense_order"]] if "dense_order" in d else sorted(dn_all)
    dense = {b: dn_all[b] for b in order}
    coeffs = {int(b): CoefficientPair(sx[int(b)], sy[int(b)]) for b in d["cf_ids"]}
    if rb is cb:
        cb = dict(rb)
    return UniformHMatrix(bct, ClusterBasis(rb), ClusterBasis(cb), coeffs, dense)


def save_uh(u, path, **extra) -> None:
    arrs = uh_to_arrays(u)
    arrs.update({f"x_{k}": np.asarray(v) for k, v in extra.items()})
    np.savez_compressed(path, **arrs)


def load_uh(path):
    """Returns (UniformHMatrix mirror, dict of extra arrays saved with ``save_uh``)."""
    with np.load(path) as z:
        d = {k: z[k] for k in z.files}
    extra = {k[2:]: v for k, v in d.items() if k.startswith("x_")}
    return uh_from_arrays(d), extra


def save_bct(bct, path, **extra) -> None:
    arrs = bct_to_arrays(bct)
    arrs["format_version"] = np.int64(FORMAT_VERSION)
    arrs.update({f"x_{k}": np.asarray(v) for k, v in extra.items()})
    np.savez_compressed(path, **arrs)


def load_bct(path):
    with np.load(path) as z:
        d = {k: z[k] for k in z.files}
    extra = {k[2:]: v for k, v in d.items() if k.startswith("x_")}
    return bct_from_arrays(d), extra


def h_to_arrays(h) -> dict:
    """HMatrix (reference hmatrix.py:39-69 or mirror) -> arrays (SVD factors + dense)."""
    out = bct_to_arrays(h.bct)
    out["format_version"] = np.int64(FORMAT_VERSION)
    ids = sorted(h.admissible)
    out["hf_ids"] = np.asarray(ids, dtype=np.int64)
    out["hu_shape"], out["hu_data"] = _pack_mats({b: h.admissible[b].U for b in ids}, ids)
    out["hv_shape"], out["hv_data"] = _pack_mats({b: h.admissible[b].V for b in ids}, ids)
    sig = [np.asarray(h.admissible[b].sigma, dtype=np.float64) for b in ids]
    out["hs_len"] = np.array([len(x) for x in sig], dtype=np.int64)
    out["hs_data"] = np.concatenate(sig) if sig else np.zeros(0)
    dids = sorted(h.dense)
    out["dn_ids"] = np.asarray(dids, dtype=np.int64)
    out["dn_shape"], out["dn_data"] = _pack_mats(h.dense, dids)
    out["dense_order"] = np.asarray(getattr(h, "_dense_order", dids), dtype=np.int64)
    return out


def h_from_arrays(d) -> HMatrix:
    bct = bct_from_arrays(d)
    ids = [int(b) for b in d["hf_ids"]]
    us = _unpack_mats(d["hf_ids"], d["hu_shape"], d["hu_data"])
    vs = _unpack_mats(d["hf_ids"], d["hv_shape"], d["hv_data"])
    off = np.concatenate([[0], np.cumsum(d["hs_len"])]).astype(np.int64)
    adm = {b: SVDForm(us[b], d["hs_data"][off[i] : off[i + 1]].copy(), vs[b]) for i, b in enumerate(ids)}
    dn_all = _unpack_mats(d["dn_ids"], d["dn_shape"], d["dn_data"])
    order = [int(b) for b in d["dense_order"]] if "dense_order" in d else sorted(dn_all)
    return HMatrix(bct, adm, {b: dn_all[b] for b in order})


def save_h(h, path, **extra) -> None:
    arrs = h_to_arrays(h)
    arrs.update({f"x_{k}": np.asarray(v) for k, v in extra.items()})
    np.savez_compressed(path, **arrs)


def load_h(path):
    with np.load(path) as z:
        d = {k: z[k] for k in z.files}
    extra = {k[2:]: v for k, v in d.items() if k.startswith("x_")}
    return h_from_arrays(d), extra
