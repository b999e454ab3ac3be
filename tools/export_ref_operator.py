"""Export a real compress-path BASELINE operator (built by the REFERENCE) to oracle/_ref/operators/.

Build container only.  Input: data/ref_cfgN.pkl (+ data/ref_cfgN_h.pkl), written by
tools/build_reference_operator.py (icosphere centroids -> assemble_h(1e-6, 1e-7) ->
compress_h_to_uh(1e-6), all in uhm_kit).  Output (git-ignored, shipped to the GPU box with
the repo snapshot, read only by tests/):

  oracle/_ref/operators/cfgN_uh.pkl   the reference's own UniformHMatrix object (unpickled on
                                       the box with uhm_kit from oracle/_ref/site)
  oracle/_ref/operators/cfgN_h.pkl    the source HMatrix (matvec_h parity), when present
  oracle/_ref/operators/cfgN_out.npz  seeded vectors and the reference's outputs computed here:
                                       uhm_kit.matvec_uh for views full / far / near (SURVEY §8c
                                       G1-G3), forward and adjoint (G4), plus matvec_h fwd/adj

usage: PYTHONPATH=oracle/_ref/site:. python tools/export_ref_operator.py CFG
"""

from __future__ import annotations

import os
import pickle
import shutil
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import uhm_kit  # noqa: E402
from matvec_oracle import farfield_only, nearfield_only  # noqa: E402

OUT = os.path.join(ROOT, "oracle", "_ref", "operators")


def main():
    cfg = int(sys.argv[1])
    os.makedirs(OUT, exist_ok=True)
    src = os.path.join(ROOT, "data", f"ref_cfg{cfg}.pkl")
    with open(src, "rb") as fh:
        d = pickle.load(fh)
    uh = d["uh"]
    with open(os.path.join(OUT, f"cfg{cfg}_uh.pkl"), "wb") as fh:
        pickle.dump(uh, fh, protocol=4)
    n_rows, n_cols = uh.shape
    rng = np.random.default_rng(0)
    xf = rng.standard_normal(n_cols) + 1j * rng.standard_normal(n_cols)  # BASELINE vector, tree order
    rng = np.random.default_rng(1)
    xa = rng.standard_normal(n_rows) + 1j * rng.standard_normal(n_rows)
    out = {"xf": xf, "xa": xa, "N": np.int64(n_rows),
           "bytes_estimate": np.int64(uhm_kit.storage_report_uh(uh).bytes_estimate)}
    t0 = time.time()
    for view, fn in (("full", lambda u: u), ("far", farfield_only), ("near", nearfield_only)):
        uv = fn(uh)
        out[f"ref_{view}_fwd"] = uhm_kit.uniform.matvec_uh(uv, xf)
        out[f"ref_{view}_adj"] = uhm_kit.uniform.matvec_uh(uv, xa, adjoint=True)
    hp = os.path.join(ROOT, "data", f"ref_cfg{cfg}_h.pkl")
    if os.path.exists(hp):
        shutil.copyfile(hp, os.path.join(OUT, f"cfg{cfg}_h.pkl"))
        with open(hp, "rb") as fh:
            h = pickle.load(fh)
        out["ref_h_fwd"] = uhm_kit.hmatrix.matvec_h(h, xf)
        out["ref_h_adj"] = uhm_kit.hmatrix.matvec_h(h, xa, adjoint=True)
    np.savez(os.path.join(OUT, f"cfg{cfg}_out.npz"), **out)
    sizes = {f: os.path.getsize(os.path.join(OUT, f)) / 1e6 for f in os.listdir(OUT) if f.startswith(f"cfg{cfg}_")}
    print(f"cfg{cfg}: N={n_rows} reference outputs in {time.time() - t0:.1f}s; files (MB) {sizes}")


if __name__ == "__main__":
    main()
