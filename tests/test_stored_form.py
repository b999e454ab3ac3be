"""Stored form of the admissible blocks (packer ``factor_bias``): factorized (s_x, s_y; the U
ops stage u_b = s_y^H y_t) iff k_b (l_s + l_t) < bias * l_s l_t, else the product S_b = s_x s_y^H.
The default is the byte minimum (bias 1) from 1 GB on and 0.5 below it (operators bound by the
forward dependency chain lose the U phase of most blocks).  Whatever the form, the product must
match the reference's stored outputs (tests/golden, written by uhm_kit itself) at 1e-12: the NumPy
VM on CPU, every engine on the GPU, forward and adjoint, single and multi RHS."""

import numpy as np
import pytest

from conftest import load_golden, rel
from packed_vm import vm_matmat, vm_matvec

NAMES = ["helm400", "ico2_helm_compress", "uh800_laplace", "rect_sphere", "degenerate"]
BIASES = [0.0, 0.5, 1.0, 1e9]  # all product ... all factorized


def _pack(u, bias):
    """bias 1.0 also runs WITHOUT the adjoint copy (partials per product block: the multi-GPU scheme)."""
    import os

    from paper_2405_15573_b200.packer import pack

    if bias != 1.0:
        return pack(u, factor_bias=bias)
    os.environ["UHMV_ADJ_COPY"] = "0"
    try:
        return pack(u, factor_bias=bias)
    finally:
        del os.environ["UHMV_ADJ_COPY"]


@pytest.mark.parametrize("name", NAMES)
def test_forms_cover_both_paths(name):
    u, _ = load_golden(name)
    f0 = _pack(u, 0.0).geo["factorized"]
    f9 = _pack(u, 1e9).geo["factorized"]
    assert not any(f0.values())
    assert sum(f9.values()) >= 0.8 * len(f9) or name == "degenerate"  # (rank-0 factors stay product)


@pytest.mark.parametrize("bias", BIASES)
@pytest.mark.parametrize("name", NAMES)
def test_stored_form_vm(name, bias):
    u, ex = load_golden(name)
    p = _pack(u, bias)
    assert rel(vm_matvec(p, ex["vf_0"]), ex["ref_fwd_0"]) <= 1e-12
    assert rel(vm_matvec(p, ex["va_0"], adjoint=True), ex["ref_adj_0"]) <= 1e-12
    W = vm_matmat(p, np.stack([ex["vf_0"], -ex["vf_0"]], axis=1))
    assert rel(W[:, 0], ex["ref_fwd_0"]) <= 1e-12 and rel(W[:, 1], -ex["ref_fwd_0"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("bias", BIASES)
@pytest.mark.parametrize("name", NAMES)
def test_stored_form_gpu(name, bias):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from conftest import ensure_built

    ensure_built()
    from paper_2405_15573_b200.device import DeviceOperator

    u, ex = load_golden(name)
    dop = DeviceOperator(_pack(u, bias), device="cuda:0")
    for adjoint, kv, kr in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
        x = torch.from_numpy(np.ascontiguousarray(ex[kv], dtype=np.complex128)).to("cuda:0")
        for mode in ("bulk", "fused"):
            assert rel(dop.matvec(x, adjoint=adjoint, mode=mode).cpu().numpy(), ex[kr]) <= 1e-12, (name, bias, adjoint, mode)
        W = dop.matmat(torch.stack([x, -x], dim=1).contiguous(), adjoint=adjoint).cpu().numpy()
        assert rel(W[:, 0], ex[kr]) <= 1e-12 and rel(W[:, 1], -ex[kr]) <= 1e-12
