"""Drop-in ``matvec_uh``: same signature and behaviour as the reference, CUDA underneath.

Reference boundary: ``matvec_uh(u, v, workers=1, adjoint=False, stats=None)``,
/root/reference/pkg/src/uhm_kit/uniform.py:476-556 (and ``UniformHMatrix.matvec``,
uniform.py:116-117).  Preserved semantics:
  * ``ValueError`` when ``v.shape != (n_in,)`` (uniform.py:493-494); 2-D input is rejected
    like the reference -- multi-RHS is the separate extension :func:`matmat_uh`;
  * result dtype ``np.result_type(v.dtype, u._dtype)`` (uniform.py:495): real operators and
    vectors are promoted to complex128 on the device (zero imaginary parts give exactly the
    real products) and the real part is returned;
  * a NEW array is returned, the input is never mutated; vectors are in tree order;
  * ``workers`` is accepted and ignored (the CUDA grid replaces the thread pool,
    _parallel.py:14-88); ``stats.count`` receives |P+| + |P-| (uniform.py:536-537, :547-548);
  * ``adjoint=True`` computes A^H v (uniform.py:498-503, :543-544).
The operator is packed once per object (cached by identity with a weakref guard) and
kept resident in HBM; every call then runs the C-ABI entry ``uhmv_matvec_host``.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np

from .device import DeviceOperator
from .packer import pack

__all__ = ["matvec_uh", "matmat_uh", "matvec_h", "matvec_uh_sym", "device_operator", "register_device_operator",
           "clear_cache"]

_cache: dict = {}
_cache_lock = threading.Lock()


def _fingerprint(u):
    if hasattr(u, "coupling"):  # SymmetricUniformHMatrix
        return (id(u.bct), id(u.basis), id(u.coupling), len(u.coupling), id(u.dense), len(u.dense), u.kind)
    if hasattr(u, "admissible"):  # HMatrix
        return (id(u.bct), id(u.admissible), len(u.admissible), id(u.dense), len(u.dense))
    return (
        id(u.bct),
        id(u.row_basis),
        id(u.col_basis),
        id(u.coeffs),
        len(u.coeffs),
        id(u.dense),
        len(u.dense),
        id(getattr(u.bct, "row_map", None)),
    )


def _pack_any(u):
    if hasattr(u, "coupling"):
        from .packer_sym import pack_sym

        return pack_sym(u)
    if hasattr(u, "admissible") and not hasattr(u, "coeffs"):
        from .packer_h import pack_h

        return pack_h(u)
    return pack(u)


def device_operator(u, device=None) -> DeviceOperator:
    """Packed, HBM-resident form of ``u`` -- a UniformHMatrix or an HMatrix (built on first
    use, then cached)."""
    key = id(u)
    fp = _fingerprint(u)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            ref, fp_old, dop = hit
            if ref() is u and fp_old == fp and (device is None or str(dop.device) == str(device)):
                return dop
        dop = DeviceOperator(_pack_any(u), device=device)
        try:
            ref = weakref.ref(u, lambda _r, k=key: _cache.pop(k, None))
        except TypeError:  # not weak-referenceable: keep it alive with the plan
            ref = (lambda obj: (lambda: obj))(u)
        _cache[key] = (ref, fp, dop)
        return dop


def register_device_operator(u, dop: DeviceOperator) -> None:
    """Use an existing DeviceOperator for ``u`` (e.g. one a benchmark or a distributed driver
    built) in every later drop-in call."""
    key = id(u)
    with _cache_lock:
        try:
            ref = weakref.ref(u, lambda _r, k=key: _cache.pop(k, None))
        except TypeError:
            ref = (lambda obj: (lambda: obj))(u)
        _cache[key] = (ref, _fingerprint(u), dop)


def clear_cache() -> None:
    with _cache_lock:
        for _ref, _fp, dop in _cache.values():
            dop.close()
        _cache.clear()


def _is_torch_cuda(v) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, torch.Tensor) and v.is_cuda


def matvec_uh(u, v, workers: int = 1, adjoint: bool = False, stats=None):
    n_rows, n_cols = u.shape
    n_in = n_rows if adjoint else n_cols
    if _is_torch_cuda(v):
        # device-resident extension: CUDA tensor in, CUDA tensor out (no host copies)
        if tuple(v.shape) != (n_in,):
            raise ValueError(f"vector of shape {tuple(v.shape)} does not match operator input size {n_in}")
        import torch

        dop = device_operator(u, device=v.device)
        out = dop.matvec(v.to(torch.complex128), adjoint=adjoint)
        if stats is not None:
            stats.count(dop.packed.n_adm + dop.packed.n_dense)
        return out
    v = np.asarray(v)
    if v.shape != (n_in,):
        raise ValueError(f"vector of shape {v.shape} does not match operator input size {n_in}")
    dtype = np.result_type(v.dtype, u._dtype)
    dop = device_operator(u)
    # pageable caller arrays go through the plan's pinned staging vectors (one host copy in,
    # the CUDA-graph host call, one copy out into the new result array)
    w = dop.matvec_array(v, adjoint=adjoint, dtype=dtype)
    if stats is not None:
        stats.count(dop.packed.n_adm + dop.packed.n_dense)
    return w


def matvec_h(h, v, workers: int = 1, adjoint: bool = False, stats=None):
    """Drop-in for the H-matrix product ``matvec_h`` (reference hmatrix.py:143-184): same
    signature, ValueError, result dtype (hmatrix.py:155-157) and stats semantics (one count
    per admissible and dense block), run on the same sm_100a engine."""
    return matvec_uh(h, v, workers=workers, adjoint=adjoint, stats=stats)


def matvec_uh_sym(us, v, workers: int = 1, adjoint: bool = False, stats=None):
    """Matvec of the symmetric single-triangle variant (symmetric.py, paper Remark 4.5) with
    the reference's ``matvec_uh`` signature and semantics (ValueError, result dtype, new array,
    stats = |P+| + |P-| of the two-triangle operator).  Every stored slab is streamed once per
    product (packer_sym).  Adjoint: the forward for a hermitian operator, conj(A conj(v)) for
    a symmetric one (A^T = A)."""
    n = us.shape[0]
    conj = bool(adjoint) and us.kind == "symmetric"
    if _is_torch_cuda(v):
        if tuple(v.shape) != (n,):
            raise ValueError(f"vector of shape {tuple(v.shape)} does not match operator input size {n}")
        import torch

        dop = device_operator(us, device=v.device)
        x = v.to(torch.complex128)
        out = dop.matvec(x.conj().resolve_conj() if conj else x)
        if stats is not None:
            stats.count(dop.packed.n_adm + dop.packed.n_dense)
        return out.conj().resolve_conj() if conj else out
    v = np.asarray(v)
    if v.shape != (n,):
        raise ValueError(f"vector of shape {v.shape} does not match operator input size {n}")
    dtype = np.result_type(v.dtype, us._dtype)
    dop = device_operator(us)
    w = dop.matvec_array(np.conj(v) if conj else v, adjoint=False, dtype=dtype)
    if stats is not None:
        stats.count(dop.packed.n_adm + dop.packed.n_dense)
    return np.conj(w) if conj else w


def matmat_uh(u, V, adjoint: bool = False):
    """Multi-RHS extension (BASELINE config 5): ``(n_in, nrhs)`` -> ``(n_out, nrhs)``.

    The reference rejects 2-D input (uniform.py:493-494); its oracle for this case is
    the column loop of single-vector calls, which is what this computes.
    """
    V = np.asarray(V)
    n_rows, n_cols = u.shape
    n_in = n_rows if adjoint else n_cols
    if V.ndim != 2 or V.shape[0] != n_in:
        raise ValueError(f"block of shape {V.shape} does not match operator input size {n_in}")
    dtype = np.result_type(V.dtype, u._dtype)
    dop = device_operator(u)
    import torch

    n_out = n_cols if adjoint else n_rows
    if V.shape[1] == 0:
        W = np.zeros((n_out, 0), np.complex128)
    else:
        X = torch.from_numpy(np.ascontiguousarray(V, dtype=np.complex128)).to(dop.device)
        W = dop.matmat(X, adjoint=adjoint).cpu().numpy()
    if np.issubdtype(dtype, np.complexfloating):
        return W.astype(dtype, copy=False)
    return W.real.astype(dtype)
