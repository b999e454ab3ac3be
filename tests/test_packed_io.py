"""On-disk packed-operator format (packed_io): save -> load reproduces
every array of the arena and the programs bit for bit, and the loaded operator computes the
reference's outputs (NumPy VM of the device programs, single and multi-RHS, 1-rank and a
rank of a 2-rank partition)."""

import numpy as np
import pytest

from conftest import load_golden, rel
from packed_vm import vm_matmat, vm_matvec

from paper_2405_15573_b200.packed_io import load_packed, save_packed
from paper_2405_15573_b200.packer import MR_ROWS, pack


def _same_prog(a, b):
    for f in ("ops", "segs", "pieces", "runs", "waits", "sigs", "fused_order", "kinds", "mr_segs", "mr_ranges", "mr_lds"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert [tuple(x) for x in a.phases] == [tuple(x) for x in b.phases]
    for f in ("in_max", "xin_max", "out_max", "n_counters", "zero_output", "arena_elems", "stage_elems", "w_order"):
        assert getattr(a, f) == getattr(b, f), f
    assert (a.part_b is None) == (b.part_b is None)
    if a.part_b is not None:
        _same_prog(a.part_b, b.part_b)


@pytest.mark.parametrize("name", ["helm400", "ico2_helm_compress", "rect_sphere", "no_admissible"])
def test_roundtrip_and_parity(name, tmp_path):
    u, ex = load_golden(name)
    p = pack(u)
    path = str(tmp_path / "op.npz")
    save_packed(path, p)
    q = load_packed(path)
    assert np.array_equal(p.arena, q.arena) and q.arena.dtype == np.complex128
    _same_prog(p.fwd, q.fwd)
    _same_prog(p.adj, q.adj)
    key = (MR_ROWS, MR_ROWS)
    assert key in q.rechunked and q.geo is None
    for a, b in zip(p.rechunked[key][:2], q.rechunked[key][:2]):
        _same_prog(a, b)
    assert (q.n_rows, q.n_cols, q.work_len, q.bytes_alg) == (p.n_rows, p.n_cols, p.work_len, p.bytes_alg)
    # the loaded pack computes the reference's outputs
    for adjoint, vk, rk in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
        w = vm_matvec(q, ex[vk], adjoint=adjoint, order="fused", engine="pieces")
        assert rel(w, ex[rk]) <= 1e-12
    rng = np.random.default_rng(1)
    V = rng.standard_normal((q.n_cols, 3)) + 1j * rng.standard_normal((q.n_cols, 3))
    W0 = vm_matmat(p, V)
    W1 = vm_matmat(q, V, programs=q.programs(rows_per_chunk=MR_ROWS, far_rows=MR_ROWS))
    assert rel(W1, W0) <= 1e-13


def test_partitioned_roundtrip(tmp_path):
    u, _ = load_golden("ico2_helm_compress")
    p = pack(u, rank=1, world=2)
    path = str(tmp_path / "r1.npz")
    save_packed(path, p)
    q = load_packed(path)
    _same_prog(p.fwd, q.fwd)
    _same_prog(p.adj, q.adj)
    assert q.world == 2 and q.rank == 1 and q.exchange == p.exchange
    assert [int(v) for v in q.part["row_bounds"]] == [int(v) for v in p.part["row_bounds"]]
    assert not q.rechunked  # multi-RHS re-chunking is single-GPU only


def test_rejects_other_files(tmp_path):
    path = str(tmp_path / "x.npz")
    np.savez(path, meta=np.array('{"format": "other"}'))
    with pytest.raises(ValueError):
        load_packed(path)
