"""BASELINE.json workloads on the GPU box, where the reference package is absent.

Each config ships as a small structure fixture ``workloads/cfgN.npz`` exported by
``tools/make_workloads.py`` from the REFERENCE's own objects (never
re-derive the tree): the cluster trees and block tree (uh_io format), the cluster ranks
l_s / l_t and block ranks k_b of the operator the reference built (configs 1-3:
icosphere centroids, ``assemble_h`` + ``compress_h_to_uh`` at 1e-6; config 4: rank 16
everywhere), plus the reference CPU timing measured in the build container.

``build_operator`` fills that structure with seeded values:
  config 4 (BASELINE.json verbatim): bases |s| x 16 orthonormal (QR of a complex Gaussian),
      S_b 16 x 16 complex Gaussian / (1 + dist_b) stored as s_x = S_b, s_y = I_16,
      dense leaves complex Gaussian;
  configs 1-3 ("rank-profile surrogate"): the same block structure and every rank of the
      reference-built Helmholtz operator, bases orthonormal, s_x / s_y / dense complex
      Gaussian.  Shapes, stored forms (per-block min of factorized vs product), bytes and
      therefore the memory traffic are identical to the real operator; only the values
      are synthetic (the real values need the reference's ACA construction).
Vectors: ``rng = default_rng(0); x = rng.standard_normal(N) + 1j*rng.standard_normal(N)``,
tree order.
"""

from __future__ import annotations

import os

import numpy as np

from .uh_io import bct_from_arrays
from .uh_types import ClusterBasis, CoefficientPair, UniformHMatrix

__all__ = ["CONFIGS", "load_structure", "build_operator", "build_symmetric_operator", "seeded_vector",
           "algorithmic_bytes", "workload_path"]

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "workloads")

CONFIGS = {
    1: dict(name="cfg1_icosphere4_helmholtz_k4", N=5120, level=4, kappa=4.0, n_min=32, kind="profile"),
    2: dict(name="cfg2_icosphere5_helmholtz_k8", N=20480, level=5, kappa=8.0, n_min=32, kind="profile"),
    3: dict(name="cfg3_icosphere6_helmholtz_k16", N=81920, level=6, kappa=16.0, n_min=64, kind="profile"),
    4: dict(name="cfg4_icosphere7_synthetic_rank16", N=327680, level=7, kappa=0.0, n_min=64, kind="rank16"),
}


def workload_path(cfg: int) -> str:
    return os.path.join(HERE, f"cfg{cfg}.npz")


def load_structure(cfg: int):
    with np.load(workload_path(cfg)) as z:
        d = {k: z[k] for k in z.files}
    bct = bct_from_arrays(d)
    return bct, d


def _aabb_dist(lo_a, hi_a, lo_b, hi_b):
    """Box distance, restating geometry.py:200-203 (zero iff the boxes intersect)."""
    gap = np.maximum(0.0, np.maximum(lo_b - hi_a, lo_a - hi_b))
    return float(np.sqrt((gap * gap).sum()))


def _orthonormal_group(rng, n, m, l):
    """n orthonormal m x l complex bases (batched QR of a complex Gaussian)."""
    if l == 0:
        return np.zeros((n, m, 0), dtype=np.complex128)
    g = rng.standard_normal((n, m, l)) + 1j * rng.standard_normal((n, m, l))
    q, _ = np.linalg.qr(g)
    return q


def _gauss(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def build_operator(cfg: int, seed: int = 0):
    """Seeded UniformHMatrix (mirror types) on the config's reference structure."""
    bct, d = load_structure(cfg)
    kind = str(d["x_kind"]) if "x_kind" in d else CONFIGS[cfg]["kind"]
    rnodes, cnodes = bct.row_tree.nodes, bct.col_tree.nodes
    rank_r, rank_c, kb = d["x_rank_row"], d["x_rank_col"], d["x_kb"]

    def bases(nodes, ids, ranks, stream):
        rng = np.random.default_rng([seed, stream])
        groups = {}
        for c in sorted(ids):
            groups.setdefault((nodes[c].size, int(ranks[c])), []).append(c)
        out = {}
        for (m, l), cs in sorted(groups.items()):
            q = _orthonormal_group(rng, len(cs), m, l)
            for i, c in enumerate(cs):
                out[c] = q[i]
        return out

    rb = bases(rnodes, bct.row_map.keys(), rank_r, 1)
    cb = bases(cnodes, bct.col_map.keys(), rank_c, 2)
    rng = np.random.default_rng([seed, 3])
    coeffs = {}
    adm = sorted(bct.admissible_leaves)
    if kind == "rank16":
        have_box = all(getattr(n, "bbox", None) is not None for n in rnodes)
        s_all = _gauss(rng, (len(adm), 16, 16))
        eye = np.eye(16, dtype=np.complex128)
        for i, b in enumerate(adm):
            blk = bct.nodes[b]
            dist = 0.0
            if have_box:
                ra, ca = rnodes[blk.row].bbox, cnodes[blk.col].bbox
                dist = _aabb_dist(ra.lo, ra.hi, ca.lo, ca.hi)
            coeffs[b] = CoefficientPair(s_all[i] / (1.0 + dist), eye)
    else:
        for b in adm:
            blk = bct.nodes[b]
            k = int(kb[b])
            ls, lt = rb[blk.row].shape[1], cb[blk.col].shape[1]
            scale = 1.0 / np.sqrt(max(k, 1))
            coeffs[b] = CoefficientPair(_gauss(rng, (ls, k)) * scale, _gauss(rng, (lt, k)))
    rng = np.random.default_rng([seed, 4])
    dense = {}
    groups = {}
    for b in bct.inadmissible_leaves:
        groups.setdefault(bct.block_shape(b), []).append(b)
    for shp, bs in sorted(groups.items()):
        vals = _gauss(rng, (len(bs),) + shp) * (1.0 / np.sqrt(shp[1]))
        for i, b in enumerate(bs):
            dense[b] = vals[i]
    dense = {b: dense[b] for b in sorted(dense)}
    return UniformHMatrix(bct, ClusterBasis(rb), ClusterBasis(cb), coeffs, dense)


def build_h_operator(cfg: int, seed: int = 0):
    """Seeded HMatrix (mirror types) with the block ranks of the H-matrix the reference
    assembled for config ``cfg`` (``assemble_h`` at 1e-6/1e-7, the source of the uniform
    compression): U_b, V_b scaled complex Gaussian, sigma_b decaying, dense leaves as
    build_operator.  Same shapes and bytes as the reference's H-matrix."""
    from .uh_types import HMatrix, SVDForm

    bct, d = load_structure(cfg)
    if "x_kb_h" not in d:
        raise ValueError(f"config {cfg} fixture has no H-matrix ranks")
    kh = d["x_kb_h"]
    rnodes, cnodes = bct.row_tree.nodes, bct.col_tree.nodes
    rng = np.random.default_rng([seed, 5])
    groups = {}
    for b in bct.admissible_leaves:
        blk = bct.nodes[b]
        groups.setdefault((rnodes[blk.row].size, cnodes[blk.col].size, int(kh[b])), []).append(b)
    adm = {}
    for (m, n, k), bs in sorted(groups.items()):
        qu = _gauss(rng, (len(bs), m, k)) / np.sqrt(max(m, 1))
        qv = _gauss(rng, (len(bs), n, k)) / np.sqrt(max(n, 1))
        for i, b in enumerate(bs):
            adm[b] = SVDForm(qu[i], np.geomspace(1.0, 1e-6, k) if k else np.zeros(0), qv[i])
    u = build_operator(cfg, seed)
    return HMatrix(bct, adm, u.dense)


def build_symmetric_operator(cfg: int, kind: str = "symmetric", seed: int = 0):
    """Seeded symmetric single-triangle variant (symmetric.py, paper Remark 4.5) on the
    config's reference structure: X_t = the row bases of ``build_operator``, the coupling of
    every lower admissible block s_x s_y^H (ell_s x ell_t, s_y fresh Gaussian), the lower dense
    leaves as stored and the diagonal ones symmetrised.  A labelled variant: not the
    reference's operator (which stores both triangles)."""
    from .symmetric import SymmetricUniformHMatrix, lower_blocks

    u = build_operator(cfg, seed)
    bct = u.bct
    low_adm, low_dense = lower_blocks(bct)
    basis = dict(u.row_basis.matrices)
    for c in bct.col_map:
        if c not in basis:
            basis[c] = np.conj(u.col_basis.matrices[c]) if kind == "symmetric" else u.col_basis.matrices[c]
    rng = np.random.default_rng([seed, 6])
    coupling = {}
    for b in low_adm:  # s_x of the block times a fresh s_y of the column cluster's (row) rank
        blk = bct.nodes[b]
        s_x = u.coeffs[b].s_x
        s_y = _gauss(rng, (basis[blk.col].shape[1], s_x.shape[1]))
        coupling[b] = s_x @ np.conj(s_y).T
    dense = {}
    for b in low_dense:
        d = u.dense[b]
        if bct.nodes[b].row == bct.nodes[b].col:
            d = 0.5 * (d + (d.T if kind == "symmetric" else np.conj(d).T))
        dense[b] = d
    return SymmetricUniformHMatrix(bct, ClusterBasis(basis), coupling, dense, kind)


def seeded_vector(n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    re = rng.standard_normal(n)
    return re + 1j * rng.standard_normal(n)


def algorithmic_bytes(packed, nrhs: int = 1) -> int:
    """operator in its cheapest stored form + one read of x + one write of w."""
    return int(packed.bytes_alg + 16 * nrhs * (packed.n_rows + packed.n_cols))
