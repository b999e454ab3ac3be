"""Export the BASELINE config structures to paper_2405_15573_b200/workloads/cfgN.npz.

Build container only (imports the reference).  Configs 1-3 read the reference-built
operators pickled by tools/build_reference_operator.py (data/ref_cfgN.pkl); config 4
builds the icosphere-7 tree and block tree with the reference (n_min=64, eta=2 weak).

Stored: the block cluster tree (uh_io format), ranks per cluster, k_b per block, the
reference's own storage_report_uh byte estimate, and the reference CPU matvec timing
and output checksums on the seeded synthetic operator of workloads.build_operator
(so the GPU box can pin its oracle at full size without the reference).

usage: PYTHONPATH=/root/reference/pkg/src:. python tools/make_workloads.py CFG [--timing]
"""

from __future__ import annotations

import hashlib
import os
import pickle
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from icosphere import icosphere_centroids  # noqa: E402

from uhm_kit import (  # noqa: E402
    AdmissibilityParams, Geometry, build_block_tree, build_cluster_tree, matvec_uh, storage_report_uh,
)

from paper_2405_15573_b200 import workloads  # noqa: E402
from paper_2405_15573_b200.uh_io import bct_to_arrays  # noqa: E402

OUT = workloads.HERE


def main():
    cfg = int(sys.argv[1])
    meta = workloads.CONFIGS[cfg]
    os.makedirs(OUT, exist_ok=True)
    extra = {}
    if cfg in (1, 2, 3):
        with open(os.path.join("data", f"ref_cfg{cfg}.pkl"), "rb") as fh:
            d = pickle.load(fh)
        uh = d["uh"]
        bct = uh.bct
        n_nodes_r = len(bct.row_tree.nodes)
        rank_r = np.full(n_nodes_r, -1, dtype=np.int64)
        rank_c = np.full(len(bct.col_tree.nodes), -1, dtype=np.int64)
        for c, m in uh.row_basis.matrices.items():
            rank_r[c] = m.shape[1]
        for c, m in uh.col_basis.matrices.items():
            rank_c[c] = m.shape[1]
        kb = np.full(len(bct.nodes), -1, dtype=np.int64)
        for b, p in uh.coeffs.items():
            kb[b] = p.s_x.shape[1]
        hp = os.path.join("data", f"ref_cfg{cfg}_h.pkl")
        if os.path.exists(hp):  # ranks of the source H-matrix (for the H-format bench)
            with open(hp, "rb") as fh:
                hsrc = pickle.load(fh)
            kh = np.full(len(bct.nodes), -1, dtype=np.int64)
            for b, f in hsrc.admissible.items():
                kh[b] = f.rank
            extra["kb_h"] = kh
        rep = storage_report_uh(uh)
        extra["ref_bytes_estimate"] = np.int64(rep.bytes_estimate)
        rng = np.random.default_rng(0)
        n = uh.shape[1]
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            y = matvec_uh(uh, x)
            ts.append(time.perf_counter() - t0)
        extra["ref_real_op_matvec_s"] = np.array(ts[1:])
        extra["ref_real_op_norm"] = np.float64(np.linalg.norm(y))
        extra["ref_real_op_sample"] = y[:: max(1, n // 512)]
    else:
        pts, w = icosphere_centroids(meta["level"])
        g = Geometry(pts, w)
        tree = build_cluster_tree(g, meta["n_min"])
        bct = build_block_tree(tree, tree, AdmissibilityParams(2.0, "weak"))
        rank_r = np.full(len(tree.nodes), -1, dtype=np.int64)
        rank_c = rank_r.copy()
        for c in bct.row_map:
            rank_r[c] = 16
        for c in bct.col_map:
            rank_c[c] = 16
        kb = np.full(len(bct.nodes), -1, dtype=np.int64)
        kb[np.asarray(bct.admissible_leaves, dtype=np.int64)] = 16
    arrs = bct_to_arrays(bct)
    perm = np.asarray(bct.row_tree.permutation, dtype=np.int64)
    arrs["x_perm_sha256"] = np.array(hashlib.sha256(perm.tobytes()).hexdigest())
    del arrs["rt_perm"]  # large; the sha pins it (uh_io regenerates identity on load)
    arrs["rt_perm"] = np.zeros(0, dtype=np.int64)
    arrs.update({f"x_{k}": v for k, v in extra.items()})
    arrs["x_rank_row"] = rank_r
    arrs["x_rank_col"] = rank_c
    arrs["x_kb"] = kb
    arrs["x_kind"] = np.array(meta["kind"])
    arrs["x_N"] = np.int64(bct.shape[0])
    path = workloads.workload_path(cfg)
    np.savez_compressed(path, **arrs)
    print(f"cfg{cfg}: wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB); "
          f"adm={len(bct.admissible_leaves)} dense={len(bct.inadmissible_leaves)}")

    # reference CPU matvec on the seeded synthetic operator (pins the oracle at full size)
    if "--timing" in sys.argv:
        u = workloads.build_operator(cfg)
        x = workloads.seeded_vector(u.shape[1], 0)
        ts = []
        y = None
        for _ in range(3):
            t0 = time.perf_counter()
            y = matvec_uh(u, x)
            ts.append(time.perf_counter() - t0)
        with np.load(path) as z:
            arrs = {k: z[k] for k in z.files}
        n = u.shape[0]
        arrs["x_ref_synth_matvec_s"] = np.array(ts)
        arrs["x_ref_synth_norm"] = np.float64(np.linalg.norm(y))
        arrs["x_ref_synth_stride"] = np.int64(max(1, n // 4096))
        arrs["x_ref_synth_sample"] = y[:: max(1, n // 4096)]
        arrs["x_ref_synth_adj_sample"] = matvec_uh(u, x, adjoint=True)[:: max(1, n // 4096)]
        np.savez_compressed(path, **arrs)
        print(f"cfg{cfg}: reference matvec on synthetic operator {min(ts):.3f}s; "
              f"norm {arrs['x_ref_synth_norm']:.6e}")


if __name__ == "__main__":
    main()
