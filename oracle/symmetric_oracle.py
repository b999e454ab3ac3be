"""CPU oracle of the symmetric single-triangle variant (paper Remark 4.5).

TEST INFRASTRUCTURE ONLY (see matvec_oracle.py header): imported by tests/ and bench.py's
CPU legs, never by the product path.

The variant is defined in paper_2405_15573_b200/symmetric.py; this is a direct block-loop
restatement of that definition, in the two-phase shape of the reference's matvec_uh
(uniform.py:509-548), extended by the mirror terms:

  phase 1: y_t = V_t^H x|_t for every cluster (V_t = conj(X_t) symmetric, X_t hermitian)
  phase 2: z_s = sum_{lower (s,t)} S_b y_t + sum_{lower (t',s)} M(S_b') y_t'   (M = ^T / ^H)
           w|_s += X_s z_s
  dense:   w|_r += D_b x|_c (lower and diagonal), w|_c += M(D_b) x|_r (strictly lower)
  adjoint: hermitian -> the forward; symmetric -> conj(A conj(x)) (A^H = conj(A) as A^T = A)

Pinned (tests/test_symmetric.py): against the REFERENCE's own matvec_uh run on the
two-triangle expansion of the same operator (tests/golden/sym_*.npz, written by
tools/make_golden_sym.py with uhm_kit), against the dense expansion, and through
A^T = A / A^H = A identities.
"""

from __future__ import annotations

import numpy as np

__all__ = ["oracle_matvec_sym", "oracle_to_dense_sym"]


def oracle_matvec_sym(us, v, adjoint: bool = False) -> np.ndarray:
    v = np.asarray(v)
    n = us.shape[0]
    if v.shape != (n,):
        raise ValueError(f"vector of shape {v.shape} does not match operator size {n}")
    dtype = np.result_type(v.dtype, us._dtype)
    if adjoint and us.kind == "symmetric":
        return np.conj(oracle_matvec_sym(us, np.conj(v))).astype(dtype, copy=False)
    bct = us.bct
    nodes = bct.row_tree.nodes
    X = us.basis.matrices
    y = {}
    for c in X:
        nd = nodes[c]
        y[c] = np.conj(us.col_basis(c)).T @ v[nd.lo : nd.hi]
    z = {c: np.zeros(X[c].shape[1], dtype=np.complex128) for c in X}
    for b, s_b in us.coupling.items():
        nd = bct.nodes[b]
        s, t = nd.row, nd.col
        z[s] += s_b @ y[t]
        z[t] += us.mirror(s_b) @ y[s]
    w = np.zeros(n, dtype=dtype)
    for c, zc in z.items():
        nd = nodes[c]
        w[nd.lo : nd.hi] += X[c] @ zc
    for b, d in us.dense.items():
        r0, r1, c0, c1 = bct.block_ranges(b)
        w[r0:r1] += d @ v[c0:c1]
        if (r0, r1) != (c0, c1):
            w[c0:c1] += us.mirror(d) @ v[r0:r1]
    return w


def oracle_to_dense_sym(us) -> np.ndarray:
    """Dense expansion (small operators only), both triangles."""
    n = us.shape[0]
    if n * n > 4_000_000:
        raise ValueError("too large to expand")
    A = np.zeros((n, n), dtype=np.complex128)
    bct = us.bct
    X = us.basis.matrices
    for b, s_b in us.coupling.items():
        r0, r1, c0, c1 = bct.block_ranges(b)
        nd = bct.nodes[b]
        blk = X[nd.row] @ s_b @ np.conj(us.col_basis(nd.col)).T
        A[r0:r1, c0:c1] = blk
        A[c0:c1, r0:r1] = us.mirror(blk)
    for b, d in us.dense.items():
        r0, r1, c0, c1 = bct.block_ranges(b)
        A[r0:r1, c0:c1] = d
        if (r0, r1) != (c0, c1):
            A[c0:c1, r0:r1] = us.mirror(d)
    return A
