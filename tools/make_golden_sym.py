"""Golden fixtures of the symmetric single-triangle variant, pinned on THE REFERENCE.

Build container only (imports uhm_kit):
    PYTHONPATH=/root/reference/pkg/src:. python tools/make_golden_sym.py

For each committed golden operator with one cluster tree (tests/golden/*.npz, built by the
reference, tools/make_golden.py) and each kind (symmetric / hermitian): the variant
``symmetrize_uh(u, kind)`` is saved (paper_2405_15573_b200.symmetric.save_sym) together with
the REFERENCE's own outputs on its two-triangle expansion -- ``expand_uh(us,
types=uhm_kit.uniform)`` is a genuine ``uhm_kit.uniform.UniformHMatrix`` whose blocks are the
variant's blocks, so ``uhm_kit.matvec_uh`` on it computes A_sym x by the reference algorithm:
  ref_fwd / ref_adj   uhm_kit.matvec_uh(expansion, v[, adjoint=True])
  dense_fwd           uhm_kit.to_dense_uh(expansion) @ v
  leaves_touched      MatvecStats count (|P+| + |P-| of the two-triangle operator)
  ref_orig_fwd        uhm_kit.matvec_uh(u, v): the operator the variant approximates
Output: tests/golden/sym_<name>_<kind>.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import uhm_kit  # noqa: E402
import uhm_kit.uniform  # noqa: E402

from paper_2405_15573_b200.symmetric import expand_uh, save_sym, symmetrize_uh  # noqa: E402
from paper_2405_15573_b200.uh_io import load_uh  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
SOURCES = ["helm400", "uh800_laplace", "ico2_helm_compress", "degenerate", "no_admissible"]


def main():
    for name in SOURCES:
        u, _ = load_uh(os.path.join(GOLD, f"{name}.npz"))
        n = u.shape[0]
        for kind in ("symmetric", "hermitian"):
            us = symmetrize_uh(u, kind)
            full = expand_uh(us, types=uhm_kit.uniform)
            assert type(full).__module__ == "uhm_kit.uniform"
            rng = np.random.default_rng(11)
            vf = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            va = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            st = uhm_kit.MatvecStats()
            out = {
                "vf": vf, "va": va,
                "ref_fwd": uhm_kit.matvec_uh(full, vf, stats=st),
                "ref_adj": uhm_kit.matvec_uh(full, va, adjoint=True),
                "ref_orig_fwd": uhm_kit.matvec_uh(u, vf),
                "leaves_touched": np.int64(st.leaves_touched),
                "bytes_estimate_two_triangle": np.int64(uhm_kit.storage_report_uh(full).bytes_estimate),
            }
            if n * n <= 4_000_000:
                out["dense_fwd"] = uhm_kit.to_dense_uh(full) @ vf
            path = os.path.join(GOLD, f"sym_{name}_{kind}.npz")
            save_sym(us, path, **out)
            print(f"{path}: {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
