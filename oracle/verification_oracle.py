"""CPU oracle: NumPy restatement of the reference power iteration.

TEST INFRASTRUCTURE ONLY (see oracle/matvec_oracle.py header).  Restates
/root/reference/pkg/src/uhm_kit/verification.py:54-85 (``_power_iteration``: power iteration
on A^H A, returns (sqrt of the Rayleigh quotient, iterations used, relative change)) and
:123-138 (``compression_error``: the same on the difference operator).  Pinned against the
reference's own values stored in tests/golden/*.npz (x_pi_*, x_ce_*).
"""

from __future__ import annotations

import math

import numpy as np

from matvec_oracle import oracle_matvec_uh

__all__ = ["power_iteration", "compression_error"]


def power_iteration(apply, apply_adjoint, n, iters, seed, stagnation=1e-6):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    rho_prev = None
    rho = 0.0
    residual = math.inf
    used = 0
    for used in range(1, iters + 1):
        w = apply(v)
        rho = float(np.real(np.vdot(w, w)))
        if rho == 0.0:
            return 0.0, used, 0.0
        z = apply_adjoint(w)
        nz = np.linalg.norm(z)
        if nz == 0.0:
            break
        v = z / nz
        if rho_prev is not None:
            residual = abs(rho - rho_prev) / rho
            if residual <= stagnation:
                break
        rho_prev = rho
    return math.sqrt(rho), used, residual


def compression_error(u_ref, u_cmp, iters=50, seed=0):
    n = u_ref.shape[1]
    norm_a, _, _ = power_iteration(
        lambda v: oracle_matvec_uh(u_ref, v), lambda v: oracle_matvec_uh(u_ref, v, adjoint=True), n, iters, seed
    )
    est, used, residual = power_iteration(
        lambda v: oracle_matvec_uh(u_ref, v) - oracle_matvec_uh(u_cmp, v),
        lambda v: oracle_matvec_uh(u_ref, v, adjoint=True) - oracle_matvec_uh(u_cmp, v, adjoint=True),
        n, iters, seed + 1,
    )
    return (est / norm_a if norm_a > 0 else est), used, residual
