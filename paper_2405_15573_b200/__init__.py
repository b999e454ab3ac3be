"""B200-native (sm_100a) uniform-H matrix-vector product, drop-in for uhm-kit's matvec_uh.

The reference (arXiv 2405.15573, package ``uhm_kit``) builds the operator; this package
packs it into HBM and replaces only the product (reference uniform.py:476-556).
"""

from .matvec import clear_cache, device_operator, matmat_uh, matvec_h, matvec_uh, matvec_uh_sym
from .packer import PackedOperator, pack
from .symmetric import SymmetricUniformHMatrix, symmetrize_uh
from .uh_types import (
    BlockClusterTree,
    BlockNode,
    Cluster,
    ClusterBasis,
    ClusterTree,
    CoefficientPair,
    HMatrix,
    MatvecStats,
    SVDForm,
    UniformHMatrix,
)

__all__ = [
    "matvec_uh",
    "matmat_uh",
    "matvec_h",
    "matvec_uh_sym",
    "SymmetricUniformHMatrix",
    "symmetrize_uh",
    "device_operator",
    "clear_cache",
    "pack",
    "PackedOperator",
    "UniformHMatrix",
    "ClusterBasis",
    "CoefficientPair",
    "ClusterTree",
    "Cluster",
    "BlockClusterTree",
    "BlockNode",
    "MatvecStats",
    "HMatrix",
    "SVDForm",
    "install",
    "uninstall",
]


def install():
    """Rebind the reference's matvec_uh names to this implementation.

    ``uhm_kit.matvec_uh`` / ``uhm_kit.uniform.matvec_uh`` (looked up at call time by
    ``UniformHMatrix.matvec``, uniform.py:117) and ``uhm_kit.verification.matvec_uh``
    (bound at import, verification.py:20); likewise ``matvec_h`` (hmatrix.py:143-184) and the
    error metrics ``spectral_norm_estimate`` / ``compression_error`` (verification.py:88-138,
    power iteration resident on the GPU for compressed operands).  Returns the originals for
    restoring.
    """
    import uhm_kit
    import uhm_kit.hmatrix
    import uhm_kit.uniform
    import uhm_kit.verification

    from . import verification as _ver

    targets = [
        (uhm_kit, "matvec_uh", matvec_uh),
        (uhm_kit.uniform, "matvec_uh", matvec_uh),
        (uhm_kit.verification, "matvec_uh", matvec_uh),
        # the H-matrix product too (hmatrix.py:143-184; HMatrix.matvec resolves it at call time)
        (uhm_kit, "matvec_h", matvec_h),
        (uhm_kit.hmatrix, "matvec_h", matvec_h),
        (uhm_kit.verification, "matvec_h", matvec_h),
        (uhm_kit, "spectral_norm_estimate", _ver.spectral_norm_estimate),
        (uhm_kit.verification, "spectral_norm_estimate", _ver.spectral_norm_estimate),
        (uhm_kit, "compression_error", _ver.compression_error),
        (uhm_kit.verification, "compression_error", _ver.compression_error),
        (_ver, "_report_cls", uhm_kit.verification.ErrorReport),
    ]
    orig = [(mod, name, getattr(mod, name)) for mod, name, _ in targets]
    for mod, name, fn in targets:
        setattr(mod, name, fn)
    return orig


def uninstall(orig) -> None:
    """Restore the bindings returned by :func:`install`."""
    for mod, name, fn in orig:
        setattr(mod, name, fn)
