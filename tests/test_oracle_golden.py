"""Pin the CPU oracle (oracle/matvec_oracle.py) against the reference's own outputs.

tests/golden/*.npz were written by tools/make_golden.py from uhm_kit itself
(/root/reference/pkg/src/uhm_kit/uniform.py:476-556); the oracle must reproduce every
stored output -- all parity views, forward and adjoint -- to 1e-12 relative l2.
"""

import numpy as np
import pytest

from conftest import rel, views
from matvec_oracle import oracle_matvec_uh, oracle_to_dense
from paper_2405_15573_b200.uh_types import MatvecStats

TOL = 1e-12


def test_oracle_matches_reference_outputs(golden):
    name, u, ex = golden
    for k in range(int(ex["nvec"])):
        for vname, view, pfx in views():
            uv = view(u)
            w = oracle_matvec_uh(uv, ex[f"vf_{k}"])
            assert rel(w, ex[f"{pfx}_fwd_{k}"]) <= TOL, (name, vname, "fwd")
            w = oracle_matvec_uh(uv, ex[f"va_{k}"], adjoint=True)
            assert rel(w, ex[f"{pfx}_adj_{k}"]) <= TOL, (name, vname, "adj")


def test_oracle_dense_expansion(golden):
    name, u, ex = golden
    if "dense_fwd_0" not in ex:
        pytest.skip("no dense expansion stored")
    a = oracle_to_dense(u)
    assert rel(a @ ex["vf_0"], ex["dense_fwd_0"]) <= TOL
    assert rel(a.conj().T @ ex["va_0"], ex["dense_adj_0"]) <= TOL


def test_oracle_zero_and_stats(golden):
    name, u, ex = golden
    w = oracle_matvec_uh(u, np.zeros(u.shape[1]))
    assert not w.any() and not ex["zero_fwd"].any()
    st = MatvecStats()
    oracle_matvec_uh(u, ex["vf_0"], stats=st)
    assert st.leaves_touched == int(ex["leaves_touched"]) == len(u.coeffs) + len(u.dense)


def test_oracle_shape_error(golden):
    name, u, ex = golden
    with pytest.raises(ValueError):
        oracle_matvec_uh(u, np.zeros(u.shape[1] + 1))
    with pytest.raises(ValueError):
        oracle_matvec_uh(u, np.zeros((u.shape[1], 2)))


def test_oracle_result_dtype():
    from conftest import load_golden

    u, ex = load_golden("uh800_laplace")
    assert u._dtype == np.float64
    assert oracle_matvec_uh(u, ex["vf_0"]).dtype == np.float64
    assert oracle_matvec_uh(u, ex["vf_0"] + 0j).dtype == np.complex128


def test_power_iteration_oracle_pinned(golden):
    """oracle/verification_oracle.py reproduces the reference power iteration values."""
    from matvec_oracle import farfield_only
    from verification_oracle import compression_error, power_iteration

    name, u, ex = golden
    if "x_pi_est" not in ex and "pi_est" not in ex:
        pytest.skip("no verification values stored")
    est, used, resid = power_iteration(
        lambda v: oracle_matvec_uh(u, v), lambda v: oracle_matvec_uh(u, v, adjoint=True), u.shape[1], 30, 0
    )
    assert abs(est - float(ex["pi_est"])) <= 1e-10 * float(ex["pi_est"])
    assert used == int(ex["pi_used"])
    rel, used, resid = compression_error(u, farfield_only(u), iters=30, seed=0)
    assert abs(rel - float(ex["ce_rel"])) <= 1e-9 * float(ex["ce_rel"])
    assert used == int(ex["ce_used"])
