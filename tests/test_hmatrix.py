"""H-matrix product (reference hmatrix.py:143-184) through the same op programs.

CPU: the oracle restatement and the NumPy VM of pack_h's programs reproduce the reference's
stored matvec_h outputs (tests/golden/h_*.npz).  GPU: the sm_100a engines do too."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel
from matvec_oracle import oracle_matvec_h
from packed_vm import vm_matmat, vm_matvec
from paper_2405_15573_b200.packer_h import pack_h
from paper_2405_15573_b200.uh_io import h_from_arrays, h_to_arrays, load_h
from paper_2405_15573_b200.uh_types import MatvecStats

H_NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "h_*.npz")))
TOL = 1e-12


@pytest.fixture(params=H_NAMES, scope="module")
def hgold(request):
    h, ex = load_h(os.path.join(GOLDEN, f"{request.param}.npz"))
    return request.param, h, ex


def test_h_oracle_matches_reference(hgold):
    name, h, ex = hgold
    assert rel(oracle_matvec_h(h, ex["vf_0"]), ex["ref_fwd_0"]) <= TOL
    assert rel(oracle_matvec_h(h, ex["va_0"], adjoint=True), ex["ref_adj_0"]) <= TOL
    st = MatvecStats()
    oracle_matvec_h(h, ex["vf_0"], stats=st)
    assert st.leaves_touched == int(ex["leaves_touched"])
    with pytest.raises(ValueError):
        oracle_matvec_h(h, np.zeros(h.shape[1] + 1))


@pytest.mark.parametrize("engine", ["segs", "pieces"])
def test_h_programs_match_reference(hgold, engine):
    name, h, ex = hgold
    p = pack_h(h)
    assert rel(vm_matvec(p, ex["vf_0"], order="fused", engine=engine), ex["ref_fwd_0"]) <= TOL
    assert rel(vm_matvec(p, ex["va_0"], adjoint=True, order="fused", engine=engine), ex["ref_adj_0"]) <= TOL
    V = np.stack([ex["vf_0"], 1j * ex["vf_0"]], axis=1)
    W = vm_matmat(p, V)
    assert rel(W[:, 0], ex["ref_fwd_0"]) <= TOL and rel(W[:, 1], 1j * ex["ref_fwd_0"]) <= TOL


def test_h_io_round_trip(hgold):
    name, h, ex = hgold
    g = h_from_arrays(h_to_arrays(h))
    assert sorted(g.admissible) == sorted(h.admissible) and sorted(g.dense) == sorted(h.dense)
    for b, f in h.admissible.items():
        assert np.array_equal(g.admissible[b].U, f.U) and np.array_equal(g.admissible[b].sigma, f.sigma)
    assert g._adm_order == h._adm_order


@pytest.mark.gpu
def test_h_matvec_on_device(hgold):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_15573_b200 as pk
    from conftest import ensure_built

    ensure_built()
    name, h, ex = hgold
    st = MatvecStats()
    w = pk.matvec_h(h, ex["vf_0"], stats=st)
    assert w.dtype == np.result_type(ex["vf_0"].dtype, h._dtype)
    assert rel(w, ex["ref_fwd_0"]) <= TOL
    assert st.leaves_touched == int(ex["leaves_touched"])
    assert rel(pk.matvec_h(h, ex["va_0"], adjoint=True), ex["ref_adj_0"]) <= TOL
    dop = pk.device_operator(h)
    for mode in ("phased", "fused", "bulk"):
        x = torch.from_numpy(np.asarray(ex["vf_0"], dtype=np.complex128)).cuda()
        assert rel(dop.matvec(x, mode=mode).cpu().numpy(), ex["ref_fwd_0"]) <= TOL
