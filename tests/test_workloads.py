"""BASELINE config workloads: structure fixtures and the seeded synthetic operators.

The reference's own matvec on the same seeded operator was recorded in the build
container (tools/make_workloads.py --timing); the oracle must reproduce those samples.
"""

import os

import numpy as np
import pytest

from conftest import rel
from matvec_oracle import oracle_matvec_uh
from paper_2405_15573_b200 import workloads
from paper_2405_15573_b200.packer import pack


def _available(cfg):
    return os.path.exists(workloads.workload_path(cfg))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_structure_fixture(cfg):
    if not _available(cfg):
        pytest.skip("fixture not generated")
    bct, d = workloads.load_structure(cfg)
    meta = workloads.CONFIGS[cfg]
    assert bct.shape == (meta["N"], meta["N"])
    leaves = [n for n in bct.row_tree.nodes if n.is_leaf]
    assert sum(n.size for n in leaves) == meta["N"]
    assert all(meta["n_min"] <= n.size <= 2 * meta["n_min"] for n in leaves)
    # every admissible block pairs clusters of equal level in these configs
    for b in bct.admissible_leaves[:2000]:
        blk = bct.nodes[b]
        assert bct.row_tree.nodes[blk.row].level == bct.col_tree.nodes[blk.col].level
    assert (d["x_kb"][np.asarray(bct.admissible_leaves)] >= 0).all()


@pytest.mark.parametrize("cfg", [1, 2])
def test_synthetic_operator_matches_reference_samples(cfg):
    if not _available(cfg):
        pytest.skip("fixture not generated")
    u = workloads.build_operator(cfg)
    bct, d = workloads.load_structure(cfg)
    if "x_ref_synth_sample" not in d:
        pytest.skip("no reference samples")
    x = workloads.seeded_vector(u.shape[1], 0)
    w = oracle_matvec_uh(u, x)
    stride = int(d["x_ref_synth_stride"])
    assert rel(w[::stride], d["x_ref_synth_sample"]) <= 1e-12
    assert abs(np.linalg.norm(w) - float(d["x_ref_synth_norm"])) <= 1e-12 * float(d["x_ref_synth_norm"])
    wa = oracle_matvec_uh(u, x, adjoint=True)
    assert rel(wa[::stride], d["x_ref_synth_adj_sample"]) <= 1e-12


def test_cfg1_bytes_match_survey():
    if not _available(1):
        pytest.skip("fixture not generated")
    p = pack(workloads.build_operator(1))
    b = workloads.algorithmic_bytes(p)
    assert 95e6 < b < 104e6  # ~99.2 MB (small drift allowed, hazard H2)
