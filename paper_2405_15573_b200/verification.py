"""Device-resident power iteration over the CUDA matvec.

The reference's error metrics (``verification.py:54-138``: ``_power_iteration``,
``spectral_norm_estimate``, ``compression_error``) call forward and adjoint matvecs up to
2 x 50 times with host vectors.  Here the iterate stays in HBM: each step is two launches of
the sm_100a kernels (forward, adjoint) plus two device reductions; only the Rayleigh
quotient crosses to the host for the stagnation test.  Semantics (seeded real start vector,
stagnation rule, return values) follow the reference line by line.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["ErrorReport", "power_iteration", "spectral_norm_estimate", "compression_error"]


@dataclass
class ErrorReport:
    """Mirror of the reference ``ErrorReport`` (verification.py:32-39)."""

    rel_spectral_estimate: float
    iterations: int
    residual: float
    frobenius_components: dict | None = None


def power_iteration(apply, apply_adjoint, n, iters, seed, stagnation=1e-6, device=None):
    """Power iteration on A^H A with device closures (restates verification.py:54-85)."""
    import torch

    rng = np.random.default_rng(seed)
    v0 = rng.standard_normal(n)
    v0 /= np.linalg.norm(v0)
    v = torch.from_numpy(v0.astype(np.complex128)).to(device)
    rho_prev = None
    rho = 0.0
    residual = math.inf
    used = 0
    for used in range(1, iters + 1):
        w = apply(v)
        rho = float(torch.vdot(w, w).real.item())
        if rho == 0.0:
            return 0.0, used, 0.0
        z = apply_adjoint(w)
        nz = float(torch.linalg.vector_norm(z).item())
        if nz == 0.0:
            break
        v = z / nz
        if rho_prev is not None:
            residual = abs(rho - rho_prev) / rho
            if residual <= stagnation:
                break
        rho_prev = rho
    return math.sqrt(rho), used, residual


def _closures(u, device=None):
    from .matvec import device_operator

    dop = device_operator(u, device=device)
    return (lambda v: dop.matvec(v)), (lambda v: dop.matvec(v, adjoint=True)), u.shape[1], dop.device


def spectral_norm_estimate(u, iters: int = 50, seed: int = 0, device=None) -> float:
    """Largest-singular-value estimate of a UniformHMatrix (verification.py:88-99)."""
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    ap, aa, n, dev = _closures(u, device)
    est, _, _ = power_iteration(ap, aa, n, iters, seed, device=dev)
    return est


def compression_error(u_ref, u_cmp, iters: int = 50, seed: int = 0, device=None) -> ErrorReport:
    """||A_ref - A_cmp||_2 / ||A_ref||_2 for two UniformHMatrix (verification.py:123-138)."""
    ap, aa, n, dev = _closures(u_ref, device)
    bp, ba, n_cmp, _ = _closures(u_cmp, dev)
    if n != n_cmp:
        raise ValueError(f"operator input sizes differ: {n} vs {n_cmp}")
    norm_a, _, _ = power_iteration(ap, aa, n, iters, seed, device=dev)
    est, used, residual = power_iteration(
        lambda v: ap(v) - bp(v), lambda v: aa(v) - ba(v), n, iters, seed + 1, device=dev
    )
    rel = est / norm_a if norm_a > 0 else est
    return ErrorReport(rel_spectral_estimate=rel, iterations=used, residual=residual)
