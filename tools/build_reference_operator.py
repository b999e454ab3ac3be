"""Build a BASELINE config operator with the REFERENCE package (this container only).

Construction stays in the reference:
icosphere centroids -> Geometry -> build_cluster_tree -> build_block_tree(eta=2, weak)
-> EntryOracle(helmholtz, kappa) -> assemble_h(1e-6, 1e-7) -> compress_h_to_uh(1e-6).
The result is pickled under data/ (git- and gpurun-ignored) for fixture extraction.

usage: PYTHONPATH=/root/reference/pkg/src python tools/build_reference_operator.py CFG
"""

import pickle
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from icosphere import icosphere_centroids  # noqa: E402

from uhm_kit import (  # noqa: E402
    AdmissibilityParams, EntryOracle, Geometry, KernelSpec, ToleranceSpec,
    assemble_h, build_block_tree, build_cluster_tree, compress_h_to_uh,
)

CONFIGS = {1: (4, 4.0, 32), 2: (5, 8.0, 32), 3: (6, 16.0, 64)}


def main():
    cfg = int(sys.argv[1])
    level, kappa, n_min = CONFIGS[cfg]
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    t0 = time.time()
    pts, w = icosphere_centroids(level)
    g = Geometry(pts, w, label=f"icosphere{level}")
    tree = build_cluster_tree(g, n_min)
    bct = build_block_tree(tree, tree, AdmissibilityParams(2.0, "weak"))
    oracle = EntryOracle(g, g, KernelSpec("helmholtz", kappa), tree.permutation, tree.permutation)
    t1 = time.time()
    h = assemble_h(oracle, bct, ToleranceSpec(1e-6), ToleranceSpec(1e-7), workers=workers)
    t2 = time.time()
    uh = compress_h_to_uh(h, 1e-6)
    t3 = time.time()
    print(f"cfg{cfg}: N={len(g)} tree+bct {t1-t0:.1f}s assemble_h {t2-t1:.1f}s compress {t3-t2:.1f}s", flush=True)
    with open(f"data/ref_cfg{cfg}.pkl", "wb") as fh:
        pickle.dump({"uh": uh, "points": pts, "weights": w, "h_matvec_ok": True}, fh, protocol=4)
    with open(f"data/ref_cfg{cfg}_h.pkl", "wb") as fh:
        pickle.dump(h, fh, protocol=4)


if __name__ == "__main__":
    main()
