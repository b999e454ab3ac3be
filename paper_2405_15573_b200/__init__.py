"""B200-native (sm_100a) uniform-H matrix-vector product, drop-in for uhm-kit's matvec_uh.

The reference (arXiv 2405.15573, package ``uhm_kit``) builds the operator; this package
packs it into HBM and replaces only the product (reference uniform.py:476-556).
"""

from .matvec import clear_cache, device_operator, matmat_uh, matvec_uh
from .packer import PackedOperator, pack
from .uh_types import (
    BlockClusterTree,
    BlockNode,
    Cluster,
    ClusterBasis,
    ClusterTree,
    CoefficientPair,
    MatvecStats,
    UniformHMatrix,
)

__all__ = [
    "matvec_uh",
    "matmat_uh",
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
    "install",
]


def install():
    """Rebind the reference's matvec_uh names to this implementation.

    ``uhm_kit.matvec_uh`` / ``uhm_kit.uniform.matvec_uh`` (looked up at call time by
    ``UniformHMatrix.matvec``, uniform.py:117) and ``uhm_kit.verification.matvec_uh``
    (bound at import, verification.py:20).  Returns the originals for restoring.
    """
    import uhm_kit
    import uhm_kit.uniform
    import uhm_kit.verification

    orig = (uhm_kit.matvec_uh, uhm_kit.uniform.matvec_uh, uhm_kit.verification.matvec_uh)
    uhm_kit.matvec_uh = matvec_uh
    uhm_kit.uniform.matvec_uh = matvec_uh
    uhm_kit.verification.matvec_uh = matvec_uh
    return orig
