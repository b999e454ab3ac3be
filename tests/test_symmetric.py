"""Symmetric single-triangle variant (paper Remark 4.5), CPU side.

The oracle (oracle/symmetric_oracle.py) is pinned against the REFERENCE's own matvec_uh run
on the two-triangle expansion of each variant (tests/golden/sym_*.npz, tools/make_golden_sym.py)
and against the reference's to_dense_uh; the single-triangle programs (packer_sym) are run by
the NumPy VM of the engine (oracle/packed_vm.py) and statically bounds-checked."""

import numpy as np
import pytest

from conftest import SYM_NAMES, load_golden, load_sym_golden, rel


@pytest.fixture(params=SYM_NAMES)
def sym(request):
    us, ex = load_sym_golden(request.param)
    return request.param, us, ex


def test_oracle_matches_reference_on_expansion(sym):
    from symmetric_oracle import oracle_matvec_sym

    name, us, ex = sym
    assert rel(oracle_matvec_sym(us, ex["vf"]), ex["ref_fwd"]) <= 1e-12, name
    assert rel(oracle_matvec_sym(us, ex["va"], adjoint=True), ex["ref_adj"]) <= 1e-12, name
    if "dense_fwd" in ex:
        assert rel(oracle_matvec_sym(us, ex["vf"]), ex["dense_fwd"]) <= 1e-12, name


def test_dense_expansion_is_symmetric(sym):
    from symmetric_oracle import oracle_to_dense_sym

    _name, us, _ex = sym
    A = oracle_to_dense_sym(us)
    M = A.T if us.kind == "symmetric" else np.conj(A).T
    assert np.array_equal(A, M)


def test_expansion_oracle_agrees(sym):
    """The mirror-type expansion through the reference-restating oracle (matvec_oracle)."""
    from matvec_oracle import oracle_matvec_uh

    from paper_2405_15573_b200.symmetric import expand_uh

    _name, us, ex = sym
    assert rel(oracle_matvec_uh(expand_uh(us), ex["vf"]), ex["ref_fwd"]) <= 1e-12


@pytest.mark.parametrize("order", ["phased", "fused"])
def test_single_triangle_programs_vm(sym, order):
    from packed_vm import vm_matvec
    from program_check import check_packed

    from paper_2405_15573_b200.packer_sym import pack_sym

    name, us, ex = sym
    p = pack_sym(us)
    check_packed(p)
    assert p.fwd.bulk_only
    w = vm_matvec(p, ex["vf"], order=order, engine="pieces")
    assert rel(w, ex["ref_fwd"]) <= 1e-12, name
    assert p.n_adm + p.n_dense == int(ex["leaves_touched"])


def test_storage_halves(sym):
    from paper_2405_15573_b200.symmetric import storage_sym

    _name, us, ex = sym
    st = storage_sym(us)
    if st["two_triangle_total"]:
        assert st["total"] <= 0.62 * st["two_triangle_total"]
    assert 16 * st["two_triangle_total"] >= 0.9 * int(ex["bytes_estimate_two_triangle"]) - 16 * st["total"]


def test_small_groups_split_ops():
    """Tiny group caps force several Z / NEAR ops per cluster / leaf (more slot rows)."""
    from packed_vm import vm_matvec
    from symmetric_oracle import oracle_matvec_sym

    from paper_2405_15573_b200.packer_sym import pack_sym

    us, ex = load_sym_golden("sym_helm400_symmetric")
    ref = oracle_matvec_sym(us, ex["vf"])
    for cap in (1, 16, 64):
        p = pack_sym(us, group_out=cap)
        assert rel(vm_matvec(p, ex["vf"], order="fused", engine="pieces"), ref) <= 1e-12


def test_two_tree_operator_rejected():
    from paper_2405_15573_b200.symmetric import symmetrize_uh

    u, _ = load_golden("two_cloud")
    with pytest.raises(ValueError):
        symmetrize_uh(u)


def test_save_load_roundtrip(tmp_path):
    from paper_2405_15573_b200.symmetric import load_sym, save_sym

    us, _ = load_sym_golden("sym_ico2_helm_compress_hermitian")
    save_sym(us, tmp_path / "s.npz")
    us2, _ = load_sym(tmp_path / "s.npz")
    assert us2.kind == us.kind and set(us2.coupling) == set(us.coupling)
    for b in us.coupling:
        assert np.array_equal(us.coupling[b], us2.coupling[b])
    for c in us.basis.matrices:
        assert np.array_equal(us.basis.matrices[c], us2.basis.matrices[c])


def test_variant_close_to_helmholtz_operator():
    """helm400's kernel matrix is symmetric up to its quadrature weights: the variant moves
    its product only at the compression tolerance level."""
    us, ex = load_sym_golden("sym_helm400_symmetric")
    assert rel(ex["ref_fwd"], ex["ref_orig_fwd"]) < 1e-8
