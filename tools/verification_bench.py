"""The reference's error metric at config 3: uhm_kit.verification.compression_error
(verification.py:123-138; power iteration :54-85) of the config-3 operator against its own
farfield-only view, three ways, same iterations and seed:
  reference      the unmodified reference loop, CPU matvecs (bounded: --ref-iters)
  installed      the reference loop after paper_2405_15573_b200.install(): host vectors, every
                 matvec through the CUDA drop-in (the H2D / D2H copies of every call included)
  device         paper_2405_15573_b200.verification.compression_error: the iterate stays in HBM
usage (GPU box, reference in oracle/_ref/site): python tools/verification_bench.py [iters]
Prints one JSON line."""

import json
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.append(os.path.join(ROOT, "oracle", "_ref", "site"))

import uhm_kit.verification as refver  # noqa: E402
from matvec_oracle import farfield_only  # noqa: E402

import paper_2405_15573_b200 as pk  # noqa: E402
from paper_2405_15573_b200 import verification as ours  # noqa: E402
from paper_2405_15573_b200 import workloads  # noqa: E402


def as_reference(u):
    """The mirror-type operator as the reference's own UniformHMatrix (verification.py:101-120
    dispatches on isinstance)."""
    import uhm_kit.uniform as U

    coeffs = {b: U.CoefficientPair(p.s_x, p.s_y) for b, p in u.coeffs.items()}
    return U.UniformHMatrix(u.bct, U.ClusterBasis(dict(u.row_basis.matrices)), U.ClusterBasis(dict(u.col_basis.matrices)),
                            coeffs, dict(u.dense))


def timed(fn):
    t = time.perf_counter()
    r = fn()
    return r, time.perf_counter() - t


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    ref_iters = int(os.environ.get("REF_ITERS", "3"))
    cfg = int(os.environ.get("CFG", "3"))
    u = as_reference(workloads.build_operator(cfg))
    far = farfield_only(u)
    res = {"config": cfg, "iters": iters, "seed": 0}
    ours.compression_error(u, far, iters=2, seed=0)  # pack + plan both operands (untimed)
    dev, t_dev = timed(lambda: ours.compression_error(u, far, iters=iters, seed=0))
    orig = pk.install()
    try:
        pk.matvec_uh(u, workloads.seeded_vector(u.shape[1], 0))
        inst, t_inst = timed(lambda: refver.compression_error(u, far, iters=iters, seed=0))
    finally:
        pk.uninstall(orig)
    cpu, t_cpu = timed(lambda: refver.compression_error(u, far, iters=ref_iters, seed=0))
    cpu_dev, _ = timed(lambda: ours.compression_error(u, far, iters=ref_iters, seed=0))
    res.update({
        "device": {"s": t_dev, "rel": dev.rel_spectral_estimate, "iterations": dev.iterations, "residual": dev.residual},
        "installed_reference_loop": {"s": t_inst, "rel": inst.rel_spectral_estimate, "iterations": inst.iterations},
        "reference_cpu": {"s": t_cpu, "iters_run": ref_iters, "rel": cpu.rel_spectral_estimate,
                          "iterations": cpu.iterations, "s_per_iteration": t_cpu / max(cpu.iterations, 1)},
        "device_vs_reference_cpu_same_iters_rel_diff": abs(cpu_dev.rel_spectral_estimate - cpu.rel_spectral_estimate)
        / abs(cpu.rel_spectral_estimate),
        "device_vs_installed_rel_diff": abs(dev.rel_spectral_estimate - inst.rel_spectral_estimate)
        / abs(inst.rel_spectral_estimate),
    })
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
