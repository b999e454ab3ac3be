"""Run each engine once per golden operator (and config 1) for compute-sanitizer.

usage (GPU box):  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \
                      python tools/sanitize.py ENGINE [--cfg1]
ENGINE: bulk | io | peer | mrtc | fused | phased.  Each run is checked against the CPU oracle
(test infrastructure) so a sanitizer-clean run is also a correct one.  Small on purpose: the
sanitizer slows the kernels 10-1000x.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402
from matvec_oracle import oracle_matvec_uh  # noqa: E402  (checker only)

from paper_2405_15573_b200.device import DeviceOperator  # noqa: E402
from paper_2405_15573_b200.packer import pack  # noqa: E402
from paper_2405_15573_b200.uh_io import load_uh  # noqa: E402

GOLD = ["helm400", "uh800_laplace", "degenerate", "rect_sphere", "ico2_helm_compress"]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run(u, engine, name):
    dev = torch.device("cuda", 0)
    worst = 0.0
    if engine == "peer":
        from paper_2405_15573_b200.dist import PeerEmulation

        em = PeerEmulation(u, 2, device=dev)
    else:
        dop = DeviceOperator(pack(u), device=dev)
    for adjoint in (False, True):
        n_in = u.shape[0] if adjoint else u.shape[1]
        rng = np.random.default_rng(3)
        v = rng.standard_normal(n_in) + 1j * rng.standard_normal(n_in)
        ref = oracle_matvec_uh(u, v, adjoint=adjoint)
        if engine in ("bulk", "fused", "phased"):
            w = dop.matvec(torch.from_numpy(v).to(dev), adjoint=adjoint, mode=engine).cpu().numpy()
        elif engine == "io":
            xh = torch.from_numpy(v).pin_memory()
            wh = torch.empty(len(ref), dtype=torch.complex128).pin_memory()
            w = dop.matvec_host(xh.numpy(), adjoint=adjoint, out=wh.numpy(), host_io=True).copy()
        elif engine == "peer":
            w = em.matvec(torch.from_numpy(v).to(dev), adjoint=adjoint).cpu().numpy()
        elif engine == "mrtc":
            V = np.stack([v, 2 * v, v.conj()], axis=1)
            V = np.concatenate([V, rng.standard_normal((n_in, 13)) + 0j], axis=1)
            W = dop.matmat(torch.from_numpy(np.ascontiguousarray(V)).to(dev), adjoint=adjoint).cpu().numpy()
            w = W[:, 0]
            worst = max(worst, rel(W[:, 1], 2 * ref))
        else:
            raise SystemExit(f"unknown engine {engine}")
        worst = max(worst, rel(w, ref))
    torch.cuda.synchronize()
    print(f"{engine} {name}: max rel err {worst:.2e}", flush=True)
    assert worst <= 1e-12, (engine, name, worst)


def main():
    engine = sys.argv[1]
    for g in GOLD:
        u, _ = load_uh(os.path.join(ROOT, "tests", "golden", f"{g}.npz"))
        run(u, engine, g)
    if "--cfg1" in sys.argv:
        from paper_2405_15573_b200 import workloads

        run(workloads.build_operator(1), engine, "cfg1")
    print("sanitize run ok", flush=True)


if __name__ == "__main__":
    main()
