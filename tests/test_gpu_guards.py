"""Out-of-bounds write detection on the device (compute-sanitizer is closed on this GPU pool,
profiles/r02/sanitizer_closed.txt).  Every buffer the kernels write -- work, dependency
counters, ticket / exit counters, host-call scratch vectors, the multi-RHS work block and the
outputs -- sits between 4096-element sentinel bands (DeviceOperator(guard=...)); each engine
runs forward and adjoint on every golden operator, config 1 and the symmetric variant, and
the bands must come back bit-identical, with the results at 1e-12 of the CPU oracle.  Reads
out of bounds are covered statically by oracle/program_check.py (tests/test_program_bounds.py)."""

import numpy as np
import pytest

from conftest import GOLDEN_NAMES, ensure_built, load_golden, load_sym_golden, rel

pytestmark = pytest.mark.gpu
G = 4096


@pytest.fixture(scope="module", autouse=True)
def _lib():
    ensure_built()


def _run_all(u, dop, oracle):
    import torch

    for adjoint in (False, True):
        n_in, n_out = (u.shape[0], u.shape[1]) if adjoint else (u.shape[1], u.shape[0])
        rng = np.random.default_rng(5)
        v = rng.standard_normal(n_in) + 1j * rng.standard_normal(n_in)
        ref = oracle(u, v, adjoint)
        x = dop.zeros(n_in, torch.complex128)
        x.copy_(torch.from_numpy(v))
        modes = ("bulk",) if dop.progs[0].bulk_only else ("bulk", "fused", "phased")
        for mode in modes:
            out = dop.zeros(n_out, torch.complex128)
            dop.matvec(x, adjoint=adjoint, mode=mode, out=out)
            assert rel(out.cpu().numpy(), ref) <= 1e-12, (mode, adjoint)
        w = dop.matvec_host(np.ascontiguousarray(v), adjoint=adjoint, host_io=False)
        assert rel(w, ref) <= 1e-12
        if not dop.progs[0].bulk_only:
            X = torch.from_numpy(np.stack([v] * 16, axis=1)).cuda()
            W = dop.matmat(X, adjoint=adjoint).cpu().numpy()
            assert rel(W[:, 3], ref) <= 1e-12
    assert dop.check_guards() == []


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_guards_golden(name):
    from matvec_oracle import oracle_matvec_uh

    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    u, _ = load_golden(name)
    dop = DeviceOperator(pack(u), device="cuda:0", guard=G)
    _run_all(u, dop, lambda u_, v, a: oracle_matvec_uh(u_, v, adjoint=a))
    dop.close()


def test_guards_config1():
    from matvec_oracle import oracle_matvec_uh

    from paper_2405_15573_b200 import workloads
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    u = workloads.build_operator(1)
    dop = DeviceOperator(pack(u), device="cuda:0", guard=G)
    _run_all(u, dop, lambda u_, v, a: oracle_matvec_uh(u_, v, adjoint=a))
    dop.close()


@pytest.mark.parametrize("name", ["sym_helm400_symmetric", "sym_ico2_helm_compress_hermitian"])
def test_guards_symmetric(name):
    from symmetric_oracle import oracle_matvec_sym

    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer_sym import pack_sym

    us, _ = load_sym_golden(name)
    dop = DeviceOperator(pack_sym(us), device="cuda:0", guard=G)
    # the packed pair holds the one forward program in both slots (A^H = A for hermitian; for
    # symmetric the drop-in conjugates around it), so both directions compute A v here
    _run_all(us, dop, lambda u_, v, a: oracle_matvec_sym(u_, v))
    dop.close()
