"""Symmetric single-triangle variant on the GPU (paper Remark 4.5).

Parity: the bulk engine's single-triangle programs (packer_sym, csrc/uhmv_bulk.cuh
uhmv_bulk_sym_kernel: T-mode and alias pieces) against the REFERENCE's matvec_uh on the
two-triangle expansion (tests/golden/sym_*.npz) and the CPU oracle, forward and adjoint, at
1e-12; the drop-in ``matvec_uh_sym`` (host arrays, stats); bitwise repeatability; configs 1 and
3 at full size against the oracle plus the bilinear symmetry x^T A y = y^T A x."""

import numpy as np
import pytest

from conftest import SYM_NAMES, ensure_built, load_sym_golden, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    ensure_built()


def _dop(us):
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer_sym import pack_sym

    return DeviceOperator(pack_sym(us), device="cuda:0")


@pytest.mark.parametrize("name", SYM_NAMES)
def test_sym_golden_device(name):
    import torch

    from symmetric_oracle import oracle_matvec_sym

    import paper_2405_15573_b200 as pk

    us, ex = load_sym_golden(name)
    dop = _dop(us)
    x = torch.from_numpy(ex["vf"]).cuda()
    w = dop.matvec(x).cpu().numpy()
    assert rel(w, ex["ref_fwd"]) <= 1e-12 and rel(w, oracle_matvec_sym(us, ex["vf"])) <= 1e-12, name
    w2 = dop.matvec(x).cpu().numpy()
    assert np.array_equal(w, w2)  # every w entry: two red.add addends onto zero
    with pytest.raises(RuntimeError):
        dop.matvec(x, mode="fused")  # T-mode / alias pieces: bulk engine only
    dop.close()
    st = pk.MatvecStats()
    wf = pk.matvec_uh_sym(us, ex["vf"], stats=st)
    wa = pk.matvec_uh_sym(us, ex["va"], adjoint=True)
    assert rel(wf, ex["ref_fwd"]) <= 1e-12 and rel(wa, ex["ref_adj"]) <= 1e-12, name
    assert st.leaves_touched == int(ex["leaves_touched"])
    wt = pk.matvec_uh_sym(us, torch.from_numpy(ex["va"]).cuda(), adjoint=True).cpu().numpy()
    assert rel(wt, ex["ref_adj"]) <= 1e-12
    with pytest.raises(ValueError):
        pk.matvec_uh_sym(us, ex["vf"][:-1])
    pk.clear_cache()


@pytest.mark.parametrize("cfg", [1, 3])
def test_sym_config_full_size(cfg):
    import torch

    from symmetric_oracle import oracle_matvec_sym

    from paper_2405_15573_b200 import workloads

    us = workloads.build_symmetric_operator(cfg)
    dop = _dop(us)
    n = us.shape[0]
    x = workloads.seeded_vector(n, 0)
    y = workloads.seeded_vector(n, 1)
    wx = dop.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    wy = dop.matvec(torch.from_numpy(y).cuda()).cpu().numpy()
    assert rel(wx, oracle_matvec_sym(us, x)) <= 1e-12
    # bilinear symmetry: y^T (A x) = x^T (A y) for A^T = A
    a, b = y @ wx, x @ wy
    assert abs(a - b) <= 1e-12 * max(abs(a), 1.0) * 10
    dop.close()
