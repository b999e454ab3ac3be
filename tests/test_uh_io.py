"""On-disk operator format (uh_io): round trips are bit exact."""

import numpy as np

from paper_2405_15573_b200.uh_io import uh_from_arrays, uh_to_arrays


def test_round_trip_bit_exact(golden):
    name, u, ex = golden
    v = uh_from_arrays(uh_to_arrays(u))
    assert v.shape == u.shape
    assert v._dtype == u._dtype
    assert v.bct.row_map == u.bct.row_map and v.bct.col_map == u.bct.col_map
    assert v.bct.block_of == u.bct.block_of
    assert v.bct.admissible_leaves == u.bct.admissible_leaves
    assert v.bct.inadmissible_leaves == u.bct.inadmissible_leaves
    assert v._dense_order == u._dense_order
    for b in u.bct.admissible_leaves + u.bct.inadmissible_leaves:
        assert v.bct.block_ranges(b) == u.bct.block_ranges(b)
    assert np.array_equal(v.bct.row_tree.permutation, u.bct.row_tree.permutation)
    for c, m in u.row_basis.matrices.items():
        assert np.array_equal(v.row_basis.matrices[c], m) and v.row_basis.matrices[c].dtype == m.dtype
    for c, m in u.col_basis.matrices.items():
        assert np.array_equal(v.col_basis.matrices[c], m)
    for b, p in u.coeffs.items():
        assert np.array_equal(v.coeffs[b].s_x, p.s_x) and np.array_equal(v.coeffs[b].s_y, p.s_y)
    for b, d in u.dense.items():
        assert np.array_equal(v.dense[b], d)
