"""Ordered output (opt-in ``UHMV_W_ORDER=1``, packer ``w_order``): the NEAR ops of an output
leaf store their rows of w and signal the leaf's counter, its FAR ops wait and add with a plain
read-modify-write -- no memset of w, no atomics.  Measured 1-3 % slower than memset + fp64
red.add (profiles/r02b/ab_ordered_output.txt), so it stays off by default; these tests keep the
variant correct: the NumPy VM on CPU, the bulk engine on the GPU, against the reference's stored
outputs (tests/golden, written by uhm_kit itself) at 1e-12."""

import numpy as np
import pytest

from conftest import load_golden, rel
from packed_vm import vm_matvec

NAMES = ["helm400", "ico2_helm_compress", "uh800_laplace", "rect_sphere", "degenerate", "no_admissible"]


def _pack_ordered(monkeypatch, u):
    from paper_2405_15573_b200.packer import pack

    monkeypatch.setenv("UHMV_W_ORDER", "1")
    return pack(u)


@pytest.mark.parametrize("name", NAMES)
def test_ordered_output_vm(monkeypatch, name):
    u, ex = load_golden(name)
    p = _pack_ordered(monkeypatch, u)
    assert p.fwd.w_order == (not p.fwd.zero_output) and p.adj.w_order == (not p.adj.zero_output)
    if name in ("helm400", "ico2_helm_compress", "uh800_laplace"):
        assert p.fwd.w_order and p.adj.w_order  # every leaf has nearfield: the ordered scheme applies
    assert rel(vm_matvec(p, ex["vf_0"]), ex["ref_fwd_0"]) <= 1e-12
    assert rel(vm_matvec(p, ex["va_0"], adjoint=True), ex["ref_adj_0"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_ordered_output_gpu(monkeypatch, name):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from conftest import ensure_built

    ensure_built()
    from paper_2405_15573_b200.device import DeviceOperator

    u, ex = load_golden(name)
    dop = DeviceOperator(_pack_ordered(monkeypatch, u), device="cuda:0")
    for adjoint, kv, kr in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
        x = torch.from_numpy(np.ascontiguousarray(ex[kv], dtype=np.complex128)).to("cuda:0")
        out = torch.full((len(ex[kr]),), float("nan"), dtype=torch.complex128, device="cuda:0")  # no memset runs
        w = dop.matvec(x, adjoint=adjoint, out=out).cpu().numpy()
        assert rel(w, ex[kr]) <= 1e-12, (name, adjoint)
        W = dop.matmat(torch.stack([x, 2 * x], dim=1).contiguous(), adjoint=adjoint).cpu().numpy()
        assert rel(W[:, 0], ex[kr]) <= 1e-12 and rel(W[:, 1], 2 * ex[kr]) <= 1e-12
