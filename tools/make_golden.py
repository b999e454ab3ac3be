"""Generate the committed golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Runs only in the build container (imports uhm_kit from /root/reference/pkg/src):
    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. python tools/make_golden.py

Every fixture holds a small operator built by the reference (uh_io format, readable on
the GPU box without the reference), seeded input vectors, and the reference's own
outputs for each parity view (SURVEY.md §8c gates G1-G4):
  ref_fwd_k / ref_adj_k          uhm_kit.matvec_uh(u, v_k[, adjoint=True])
  ref_far_fwd_k / ref_far_adj_k  same with dense={} (farfield only, G2)
  ref_near_fwd_k / ref_near_adj_k  same with coeffs={} and empty maps (nearfield only, G3)
  dense_fwd_k / dense_adj_k      to_dense_uh(u) @ v_k  (tests/test_uniform.py:327-348)
  leaves_touched                 MatvecStats count of one call
"""

from __future__ import annotations

import copy
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from icosphere import icosphere_centroids  # noqa: E402

import uhm_kit  # noqa: E402
from uhm_kit import (  # noqa: E402
    AdmissibilityParams, ClusterBasis, CoefficientPair, EntryOracle, Geometry, KernelSpec,
    MatvecStats, ToleranceSpec, UniformHMatrix, assemble_h, build_block_tree,
    build_cluster_tree, compress_h_to_uh, direct_build_uh, generate_sphere, matvec_uh,
    to_dense_uh,
)

from paper_2405_15573_b200.uh_io import save_h, save_uh  # noqa: E402
from uhm_kit import matvec_h, to_dense  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def far_view(u):
    c = copy.copy(u)
    c.dense = {}
    c._dense_order = []
    return c


def near_view(u):
    c = copy.copy(u)
    bct = copy.copy(u.bct)
    bct.row_map = {}
    bct.col_map = {}
    c.bct = bct
    c.coeffs = {}
    return c


def vectors(n_in_f, n_in_a, complex_, seeds):
    out = {}
    for k, s in enumerate(seeds):
        rng = np.random.default_rng(s)
        vf = rng.standard_normal(n_in_f)
        va = rng.standard_normal(n_in_a)
        if complex_:
            vf = vf + 1j * rng.standard_normal(n_in_f)
            va = va + 1j * rng.standard_normal(n_in_a)
        out[f"vf_{k}"] = vf
        out[f"va_{k}"] = va
    return out


def outputs(u, vecs, nvec, with_dense=True):
    res = {}
    far, near = far_view(u), near_view(u)
    a = to_dense_uh(u) if with_dense else None
    for k in range(nvec):
        vf, va = vecs[f"vf_{k}"], vecs[f"va_{k}"]
        res[f"ref_fwd_{k}"] = matvec_uh(u, vf)
        res[f"ref_adj_{k}"] = matvec_uh(u, va, adjoint=True)
        res[f"ref_far_fwd_{k}"] = matvec_uh(far, vf)
        res[f"ref_far_adj_{k}"] = matvec_uh(far, va, adjoint=True)
        res[f"ref_near_fwd_{k}"] = matvec_uh(near, vf)
        res[f"ref_near_adj_{k}"] = matvec_uh(near, va, adjoint=True)
        if a is not None:
            res[f"dense_fwd_{k}"] = a @ vf
            res[f"dense_adj_{k}"] = a.conj().T @ va
    st = MatvecStats()
    matvec_uh(u, vecs["vf_0"], stats=st)
    res["leaves_touched"] = np.int64(st.leaves_touched)
    res["zero_fwd"] = matvec_uh(u, np.zeros(u.shape[1]))
    return res


def verification_values(u):
    """Reference power iteration (verification.py:54-138) on the operator: the spectral norm
    estimate and the compression error against its own farfield-only view."""
    from uhm_kit.verification import _as_operator, _power_iteration, compression_error

    ap, aa, n = _as_operator(u)
    est, used, resid = _power_iteration(ap, aa, n, 30, 0)
    rep = compression_error(u, far_view(u), iters=30, seed=0)
    return {
        "pi_est": np.float64(est), "pi_used": np.int64(used), "pi_resid": np.float64(resid),
        "ce_rel": np.float64(rep.rel_spectral_estimate), "ce_used": np.int64(rep.iterations),
        "ce_resid": np.float64(rep.residual),
    }


def emit(name, u, complex_vec, seeds=(1, 2), with_dense=True, exact=None, **meta):
    vecs = vectors(u.shape[1], u.shape[0], complex_vec, seeds)
    res = outputs(u, vecs, len(seeds), with_dense)
    if len(u.coeffs) and len(u.dense):
        res.update(verification_values(u))
    if exact is not None:  # the exact kernel matrix (EntryOracle.to_dense) for the 1e-3/1e-4 pins
        for k in range(len(seeds)):
            res[f"exact_fwd_{k}"] = exact @ vecs[f"vf_{k}"]
    path = os.path.join(OUT, f"{name}.npz")
    save_uh(u, path, nvec=np.int64(len(seeds)), **vecs, **res, **meta)
    print(f"{name}: shape={u.shape} adm={len(u.coeffs)} dense={len(u.dense)} "
          f"size={os.path.getsize(path) / 1e6:.2f} MB")


def emit_h(name, h, complex_vec, seeds=(1,)):
    """H-matrix fixture: reference matvec_h outputs (hmatrix.py:143-184), fwd + adjoint."""
    vecs = vectors(h.shape[1], h.shape[0], complex_vec, seeds)
    res = {}
    for k in range(len(seeds)):
        res[f"ref_fwd_{k}"] = matvec_h(h, vecs[f"vf_{k}"])
        res[f"ref_adj_{k}"] = matvec_h(h, vecs[f"va_{k}"], adjoint=True)
    st = MatvecStats()
    matvec_h(h, vecs["vf_0"], stats=st)
    res["leaves_touched"] = np.int64(st.leaves_touched)
    path = os.path.join(OUT, f"{name}.npz")
    save_h(h, path, nvec=np.int64(len(seeds)), **vecs, **res)
    print(f"{name}: H shape={h.shape} adm={len(h.admissible)} dense={len(h.dense)} "
          f"size={os.path.getsize(path) / 1e6:.2f} MB")


def two_cloud():
    """Rectangular two-tree operator (tests/test_uniform.py:45-60 geometry)."""
    rng = np.random.default_rng(0)
    row_pts = rng.uniform(-0.05, 0.05, (60, 3))
    col_pts = np.concatenate([
        rng.uniform(-0.5, 0.5, (20, 3)) + np.array([10.0, 0, 0]),
        rng.uniform(-0.5, 0.5, (20, 3)) + np.array([30.0, 0, 0]),
    ])
    row_g, col_g = Geometry(row_pts, np.ones(60)), Geometry(col_pts, np.ones(40))
    row_t = build_cluster_tree(row_g, n_min=60)
    col_t = build_cluster_tree(col_g, n_min=10)
    bct = build_block_tree(row_t, col_t, AdmissibilityParams(1.0, "strong"))
    oracle = EntryOracle(row_g, col_g, KernelSpec("helmholtz", 1.0), row_t.permutation, col_t.permutation)
    return direct_build_uh(oracle, bct, 1e-8)


def rect_sphere():
    """Rectangular operator with two different sphere trees (blocks of unequal levels)."""
    g_r = generate_sphere(300, 1.0, seed=3)
    pts = generate_sphere(180, 1.0, seed=4).points * 1.7
    g_c = Geometry(pts, np.full(180, 0.05))
    t_r = build_cluster_tree(g_r, 12)
    t_c = build_cluster_tree(g_c, 20)
    bct = build_block_tree(t_r, t_c, AdmissibilityParams(2.0, "weak"))
    oracle = EntryOracle(g_r, g_c, KernelSpec("helmholtz", 3.0), t_r.permutation, t_c.permutation)
    return direct_build_uh(oracle, bct, 1e-6)


def degenerate(u):
    """Edge cases the reference accepts: rank-0 blocks, l=0 bases."""
    rb = {c: m.copy() for c, m in u.row_basis.matrices.items()}
    cb = {c: m.copy() for c, m in u.col_basis.matrices.items()}
    coeffs = {b: CoefficientPair(p.s_x.copy(), p.s_y.copy()) for b, p in u.coeffs.items()}
    rids, cids = sorted(rb), sorted(cb)
    for c in rids[::5]:  # zero-width row bases
        rb[c] = rb[c][:, :0]
    for c in cids[1::7]:  # zero-width column bases
        cb[c] = cb[c][:, :0]
    for i, b in enumerate(sorted(coeffs)):
        blk = u.bct.nodes[b]
        lr, lc = rb[blk.row].shape[1], cb[blk.col].shape[1]
        k = 0 if i % 4 == 0 else coeffs[b].s_x.shape[1]
        rng = np.random.default_rng(b)
        coeffs[b] = CoefficientPair(
            rng.standard_normal((lr, k)) + 1j * rng.standard_normal((lr, k)),
            rng.standard_normal((lc, k)) + 1j * rng.standard_normal((lc, k)),
        )
    return UniformHMatrix(u.bct, ClusterBasis(rb), ClusterBasis(cb), coeffs, dict(u.dense))


def main():
    os.makedirs(OUT, exist_ok=True)
    from conftest import Instance  # reference test fixture (tests/conftest.py:14-34)

    inst = Instance(800)
    uh800 = direct_build_uh(inst.oracle, inst.bct, 1e-4, workers=2)
    emit("uh800_laplace", uh800, complex_vec=False, seeds=(2, 4), exact=inst.dense)

    helm = Instance(400, kernel="helmholtz", kappa=2.0)
    uh400 = direct_build_uh(helm.oracle, helm.bct, 1e-5)
    emit("helm400", uh400, complex_vec=True, seeds=(5,), exact=helm.dense)
    h800 = assemble_h(inst.oracle, inst.bct, ToleranceSpec(1e-4 / 3), ToleranceSpec(1e-5), workers=2)
    emit_h("h_h800_laplace", h800, complex_vec=False, seeds=(3,))

    # configs' construction at small scale: icosphere L=2 centroids, eta=2 weak, compress path
    pts, w = icosphere_centroids(2)
    g = Geometry(pts, w)
    tree = build_cluster_tree(g, 8)
    bct = build_block_tree(tree, tree, AdmissibilityParams(2.0, "weak"))
    oracle = EntryOracle(g, g, KernelSpec("helmholtz", 2.0), tree.permutation, tree.permutation)
    h = assemble_h(oracle, bct, ToleranceSpec(1e-6), ToleranceSpec(1e-7), workers=4)
    ico2 = compress_h_to_uh(h, 1e-6)
    emit_h("h_ico2_helm", h, complex_vec=True)
    emit("ico2_helm_compress", ico2, complex_vec=True, seeds=(0,))

    emit("two_cloud", two_cloud(), complex_vec=True, seeds=(7,))
    emit("rect_sphere", rect_sphere(), complex_vec=True, seeds=(8,))
    emit("degenerate", degenerate(uh400), complex_vec=True, seeds=(9,))

    empty = Instance(80, eta=1e-9, n_min=8)
    emit("no_admissible", direct_build_uh(empty.oracle, empty.bct, 1e-4), complex_vec=False, seeds=(10,))


if __name__ == "__main__":
    main()
