"""Reference-compatible error metrics with the power iteration resident on the GPU.

Drop-in for ``uhm_kit.verification.spectral_norm_estimate`` / ``compression_error``
(/root/reference/pkg/src/uhm_kit/verification.py:88-138; the loop is ``_power_iteration``,
:54-85): same signatures, argument meaning, return values and errors, and ``install()``
rebinds them.  Operands are what the reference's ``_as_operator`` (:101-120) accepts: an
``HMatrix``, a ``UniformHMatrix``, a dense ndarray or an ``(apply, apply_adjoint, n)`` triple.

* When every operand is an H / uniform-H matrix or a dense array, the iterate never leaves HBM:
  each step is a forward and an adjoint launch of the sm_100a engine per compressed operand
  (a cuBLAS GEMV for a dense one) and two device reductions.  The host only reads the two
  scalars (rho, ||z||) it needs for the stagnation test -- one pinned copy per step, read one
  step late: step i+1 is already enqueued when step i's scalars are examined, so the GPU never
  idles on the host (the speculative last step is discarded; results are those of the
  reference's loop).
* With a Python-closure operand the loop runs on host vectors exactly as the reference does
  (compressed operands then use the host drop-in ``matvec_uh`` / ``matvec_h``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["ErrorReport", "power_iteration", "spectral_norm_estimate", "compression_error", "operator_norm_estimate"]


@dataclass
class ErrorReport:
    """Mirror of the reference ``ErrorReport`` (verification.py:32-39); after ``install()``
    the reference's own class is returned instead."""

    rel_spectral_estimate: float
    iterations: int
    residual: float
    frobenius_components: dict | None = None


_report_cls = ErrorReport  # install() points this at uhm_kit.verification.ErrorReport


def _is_compressed(a) -> bool:
    return hasattr(a, "bct") and (hasattr(a, "coeffs") or hasattr(a, "admissible"))


def _start_vector(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    return v / np.linalg.norm(v)


def _host_power_iteration(apply, apply_adjoint, n, iters, seed, stagnation=1e-6):
    """Host-vector loop, step for step verification.py:54-85 (closure operands)."""
    v = _start_vector(n, seed)
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


def power_iteration(apply, apply_adjoint, n, iters, seed, stagnation=1e-6, device=None):
    """verification.py:54-85 with DEVICE closures (CUDA complex128 tensors in and out): the
    same iterates, stagnation rule and return values, one host read per step, lagged by one
    step (see the module docstring)."""
    import torch

    v = torch.from_numpy(_start_vector(n, seed).astype(np.complex128)).to(device)

    def launch(v):
        w = apply(v)
        rho_t = torch.vdot(w, w).real
        z = apply_adjoint(w)
        nz_t = torch.linalg.vector_norm(z)
        host = torch.empty(2, dtype=torch.float64, pin_memory=True)
        host.copy_(torch.stack([rho_t, nz_t]), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return host, ev, z / nz_t

    rho_prev = None
    rho = 0.0
    residual = math.inf
    used = 0
    cur = launch(v)
    for used in range(1, iters + 1):
        nxt = launch(cur[2]) if used < iters else None  # speculative: discarded if we stop here
        host, ev, _v = cur
        ev.synchronize()
        rho, nz = host.tolist()
        if rho == 0.0:
            return 0.0, used, 0.0
        if nz == 0.0:
            break
        if rho_prev is not None:
            residual = abs(rho - rho_prev) / rho
            if residual <= stagnation:
                break
        rho_prev = rho
        cur = nxt
    return math.sqrt(rho), used, residual


def _device_closures(a, device):
    """(apply, apply_adjoint, n) on CUDA tensors for a compressed or dense operand."""
    import torch

    if _is_compressed(a):
        from .matvec import device_operator

        dop = device_operator(a, device=device)
        return (lambda v: dop.matvec(v)), (lambda v: dop.matvec(v, adjoint=True)), a.shape[1]
    m = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(device)
    mh = m.conj().T.contiguous()
    return (lambda v: torch.mv(m, v)), (lambda v: torch.mv(mh, v)), a.shape[1]


def _host_closures(a):
    """verification.py:101-120 (``_as_operator``), compressed operands on the GPU drop-ins."""
    if isinstance(a, tuple) and len(a) == 3:
        return a
    if _is_compressed(a):
        from .matvec import matvec_uh

        return (lambda v: matvec_uh(a, v)), (lambda v: matvec_uh(a, v, adjoint=True)), a.shape[1]
    if isinstance(a, np.ndarray):
        return (lambda v: a @ v), (lambda v: a.conj().T @ v), a.shape[1]
    raise TypeError(f"cannot interpret {type(a).__name__} as an operator")


def _on_device(*ops) -> bool:
    return all(_is_compressed(a) or isinstance(a, np.ndarray) for a in ops) and any(_is_compressed(a) for a in ops)


def spectral_norm_estimate(apply, apply_adjoint, n: int, iters: int = 50, seed: int = 0) -> float:
    """Largest-singular-value estimate of an operator given by its action (verification.py:88-98)."""
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    est, _, _ = _host_power_iteration(apply, apply_adjoint, n, iters, seed)
    return est


def operator_norm_estimate(a, iters: int = 50, seed: int = 0, device=None) -> float:
    """``spectral_norm_estimate`` of a uniform-H / H matrix, power iteration in HBM."""
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ap, aa, n = _device_closures(a, dev)
    est, _, _ = power_iteration(ap, aa, n, iters, seed, device=dev)
    return est


def compression_error(a_ref, a_cmp, iters: int = 50, seed: int = 0):
    """Relative spectral error ||A - A_cmp||_2 / ||A||_2 (verification.py:123-138): both norms
    estimated by power iteration; operands as the reference accepts them.  Device-resident when
    no operand is a Python closure."""
    if _on_device(a_ref, a_cmp):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("compression_error on compressed operands needs a CUDA device; there is no CPU fallback")
        dev = torch.device("cuda", torch.cuda.current_device())
        ref_apply, ref_adj, n = _device_closures(a_ref, dev)
        cmp_apply, cmp_adj, n_cmp = _device_closures(a_cmp, dev)
        run = lambda f, g, s: power_iteration(f, g, n, iters, s, device=dev)  # noqa: E731
    else:
        ref_apply, ref_adj, n = _host_closures(a_ref)
        cmp_apply, cmp_adj, n_cmp = _host_closures(a_cmp)
        run = lambda f, g, s: _host_power_iteration(f, g, n, iters, s)  # noqa: E731
    if n != n_cmp:
        raise ValueError(f"operator input sizes differ: {n} vs {n_cmp}")
    norm_a, _, _ = run(ref_apply, ref_adj, seed)
    est, used, residual = run(lambda v: ref_apply(v) - cmp_apply(v), lambda v: ref_adj(v) - cmp_adj(v), seed + 1)
    rel = est / norm_a if norm_a > 0 else est
    return _report_cls(rel_spectral_estimate=rel, iterations=used, residual=residual)
