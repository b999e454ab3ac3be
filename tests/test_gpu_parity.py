"""GPU parity through the C ABI: every golden operator, parity view, direction and mode.

Gates: G1 full, G2 farfield-only, G3 nearfield-only, G4 adjoint of each --
relative l2 <= 1e-12 against the reference's stored outputs AND the CPU oracle.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden, rel, views
from matvec_oracle import oracle_matvec_uh

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from conftest import ensure_built

    ensure_built()


def _dev(u):
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    return DeviceOperator(pack(u), device="cuda:0")


@pytest.mark.parametrize("mode", ["phased", "fused", "bulk"])
def test_device_matches_reference(golden, mode):
    name, u, ex = golden
    for vname, view, pfx in views():
        uv = view(u)
        dop = _dev(uv)
        for k in range(int(ex["nvec"])):
            for adj, vkey, okey in ((False, f"vf_{k}", f"{pfx}_fwd_{k}"), (True, f"va_{k}", f"{pfx}_adj_{k}")):
                v = ex[vkey]
                x = torch.from_numpy(np.asarray(v, dtype=np.complex128)).cuda()
                w = dop.matvec(x, adjoint=adj, mode=mode).cpu().numpy()
                assert rel(w, ex[okey]) <= TOL, (name, vname, adj, mode, rel(w, ex[okey]))
                assert rel(w, oracle_matvec_uh(uv, v, adjoint=adj)) <= TOL
                assert np.isfinite(w).all()


def test_modes_bit_identical(golden):
    name, u, ex = golden
    dop = _dev(u)
    x = torch.from_numpy(np.asarray(ex["vf_0"], dtype=np.complex128)).cuda()
    a = dop.matvec(x, mode="phased").cpu().numpy()
    b = dop.matvec(x, mode="fused").cpu().numpy()
    c = dop.matvec(x, mode="fused").cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(b, c)
    d = dop.matvec(x, mode="bulk").cpu().numpy()
    e = dop.matvec(x, mode="bulk").cpu().numpy()
    assert np.array_equal(d, e)  # the bulk engine sums in its own (fixed) order
    assert np.linalg.norm(d - a) <= 1e-13 * np.linalg.norm(a)


def test_dropin_matvec_uh(golden):
    """The reference-facing call: numpy in, numpy out, reference dtype and stats semantics."""
    import paper_2405_15573_b200 as pk
    from paper_2405_15573_b200.uh_types import MatvecStats

    name, u, ex = golden
    v = ex["vf_0"]
    st = MatvecStats()
    w = pk.matvec_uh(u, v, stats=st)
    assert w.dtype == np.result_type(v.dtype, u._dtype)
    assert rel(w, ex["ref_fwd_0"]) <= TOL
    assert st.leaves_touched == int(ex["leaves_touched"])
    wa = pk.matvec_uh(u, ex["va_0"], adjoint=True, workers=8)
    assert rel(wa, ex["ref_adj_0"]) <= TOL
    z = pk.matvec_uh(u, np.zeros(u.shape[1]))
    assert not z.any()
    assert not v.flags.writeable or np.array_equal(v, ex["vf_0"])  # input untouched
    with pytest.raises(ValueError):
        pk.matvec_uh(u, np.zeros(u.shape[1] + 1))
    if "dense_fwd_0" in ex:
        assert np.linalg.norm(w - ex["dense_fwd_0"]) <= 1e-12 * np.linalg.norm(w)


def test_reference_pins_on_device():
    """tests/test_uniform.py:315-361 + test_acceptance.py:165-195 re-asserted on the GPU path."""
    import paper_2405_15573_b200 as pk

    u, ex = load_golden("uh800_laplace")
    assert not pk.matvec_uh(u, np.zeros(800)).any()
    v = ex["vf_0"]
    ref = ex["exact_fwd_0"]
    vn = v / np.linalg.norm(v)
    assert np.linalg.norm(pk.matvec_uh(u, vn) - ref / np.linalg.norm(v)) / np.linalg.norm(ref / np.linalg.norm(v)) <= 1e-3
    w = pk.matvec_uh(u, v)
    assert np.linalg.norm(w - ex["dense_fwd_0"]) <= 1e-12 * np.linalg.norm(w)
    w1 = pk.matvec_uh(u, v, workers=1)
    w8 = pk.matvec_uh(u, v, workers=8)
    assert np.linalg.norm(w1 - w8) <= 1e-12 * np.linalg.norm(w1)
    wa = pk.matvec_uh(u, ex["va_1"], adjoint=True)
    assert np.linalg.norm(wa - ex["dense_adj_1"]) <= 1e-12 * np.linalg.norm(wa)
    uc, exc = load_golden("helm400")
    wc = pk.matvec_uh(uc, exc["vf_0"])
    assert np.linalg.norm(wc - exc["exact_fwd_0"]) / np.linalg.norm(exc["exact_fwd_0"]) <= 1e-4


def test_device_tensor_api():
    import paper_2405_15573_b200 as pk

    u, ex = load_golden("helm400")
    x = torch.from_numpy(ex["vf_0"]).cuda()
    w = pk.matvec_uh(u, x)
    assert isinstance(w, torch.Tensor) and w.is_cuda
    assert rel(w.cpu().numpy(), ex["ref_fwd_0"]) <= TOL


def test_host_abi_entry():
    """uhmv_matvec_host: host buffers in/out through the C ABI."""
    u, ex = load_golden("ico2_helm_compress")
    dop = _dev(u)
    for mode in ("phased", "fused", "bulk"):
        w = dop.matvec_host(ex["vf_0"], mode=mode)
        assert rel(w, ex["ref_fwd_0"]) <= TOL
        wa = dop.matvec_host(ex["va_0"], adjoint=True, mode=mode)
        assert rel(wa, ex["ref_adj_0"]) <= TOL


@pytest.mark.parametrize("mode", ["fused", "bulk"])
def test_repeated_fused_launches_self_reset(mode):
    u, ex = load_golden("ico2_helm_compress")
    dop = _dev(u)
    x = torch.from_numpy(ex["vf_0"]).cuda()
    first = dop.matvec(x, mode=mode).cpu().numpy()
    for _ in range(50):
        w = dop.matvec(x, mode=mode)
    torch.cuda.synchronize()
    assert np.array_equal(w.cpu().numpy(), first)
    assert int(dop.counters.abs().sum()) == 0 and int(dop.ticket.item()) == 0


@pytest.mark.parametrize("engine", ["tc", "simple"])
@pytest.mark.parametrize("R", [16, 5, 64, 80])
def test_multi_rhs_dmma(golden, R, engine, monkeypatch):
    """Multi-RHS (config 5 path) on FP64 tensor cores vs the reference column loop.  ``tc``:
    the staged engine on whole-leaf programs (R = 80: two RHS passes, 64 + 16); ``simple``:
    the register engine on the single-RHS programs."""
    if engine == "simple":
        if R > 16:
            pytest.skip("register engine: cross-check at small R only")
        monkeypatch.setenv("UHMV_MRHS_ENGINE", "simple")
        monkeypatch.setenv("UHMV_MR_ROWS", "0")
    name, u, ex = golden
    dop = _dev(u)
    rng = np.random.default_rng(3)
    for adjoint in (False, True):
        n_in = u.shape[0] if adjoint else u.shape[1]
        V = rng.standard_normal((n_in, R)) + 1j * rng.standard_normal((n_in, R))
        W = dop.matmat(torch.from_numpy(V).cuda(), adjoint=adjoint).cpu().numpy()
        ref = np.stack([oracle_matvec_uh(u, V[:, j], adjoint=adjoint) for j in range(R)], axis=1)
        assert rel(W, ref) <= TOL, (name, adjoint, R, rel(W, ref))
        if R == 16:  # column j of the block == a single-vector matvec of column j
            w0 = dop.matvec(torch.from_numpy(np.ascontiguousarray(V[:, 0])).cuda(), adjoint=adjoint).cpu().numpy()
            assert rel(W[:, 0], w0) <= 1e-13


def test_power_iteration_on_device(golden):
    """Device-resident spectral norm / compression error == the reference's values."""
    from matvec_oracle import farfield_only
    from paper_2405_15573_b200 import verification

    name, u, ex = golden
    if "pi_est" not in ex:
        pytest.skip("no verification values stored")
    est = verification.operator_norm_estimate(u, iters=30, seed=0)
    assert abs(est - float(ex["pi_est"])) <= 1e-10 * float(ex["pi_est"])
    rep = verification.compression_error(u, farfield_only(u), iters=30, seed=0)
    assert abs(rep.rel_spectral_estimate - float(ex["ce_rel"])) <= 1e-9 * float(ex["ce_rel"])
    assert rep.iterations == int(ex["ce_used"])


def test_loaded_packed_operator(golden, tmp_path):
    """A packed operator saved to disk and reloaded (packed_io) runs on the device without
    the source operator: single-RHS (bulk) and multi-RHS (re-chunked programs from the file)."""
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packed_io import load_packed, save_packed
    from paper_2405_15573_b200.packer import pack

    name, u, ex = golden
    path = str(tmp_path / "op.npz")
    save_packed(path, pack(u))
    dop = DeviceOperator(load_packed(path), device="cuda:0")
    for adjoint, vk, rk in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
        x = torch.from_numpy(np.asarray(ex[vk], dtype=np.complex128)).cuda()
        assert rel(dop.matvec(x, adjoint=adjoint, mode="bulk").cpu().numpy(), ex[rk]) <= TOL
        X = torch.stack([x, 2 * x], dim=1)
        W = dop.matmat(X, adjoint=adjoint).cpu().numpy()
        assert rel(W[:, 0], ex[rk]) <= TOL and rel(W[:, 1], 2 * ex[rk]) <= TOL


@pytest.mark.parametrize("name", ["helm400", "ico2_helm_compress", "rect_sphere", "uh800_laplace", "two_cloud",
                                  "degenerate", "no_admissible"])
def test_host_io_pinned_buffers(name):
    """uhmv_matvec_host with pinned buffers: the host-I/O launch (x over PCIe in the P1 ops,
    finished output leaves drained to the host by their last NEAR / FAR op) vs the reference,
    repeated (counters self-reset) and interleaved with the pageable path."""
    import torch

    from conftest import load_golden
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    u, ex = load_golden(name)
    dop = DeviceOperator(pack(u), device="cuda:0")
    for rep in range(3):
        for adjoint, vk, rk in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
            xv = np.asarray(ex[vk], dtype=np.complex128)
            xh = torch.from_numpy(xv.copy()).pin_memory()
            n_out = len(ex[rk])
            wh = torch.full((n_out,), complex(np.nan, np.nan), dtype=torch.complex128).pin_memory()
            for host_io in (True, None):
                w = dop.matvec_host(xh.numpy(), adjoint=adjoint, out=wh.numpy(), host_io=host_io)
                assert rel(w, ex[rk]) <= 1e-12, (name, adjoint, rep)
            wp = dop.matvec_host(xv, adjoint=adjoint)  # pageable: copy path
            assert rel(wp, ex[rk]) <= 1e-12
    assert dop.attach_io() == any(q is not None for q in dop.packed.io_programs())


def test_host_call_graphs_follow_buffers():
    """The captured CUDA graph of uhmv_matvec_host is keyed by direction, buffer pair and
    path: switching between two pinned buffer pairs, pageable buffers, directions and forced
    paths in an interleaved sequence gives the reference result every time (a stale graph
    would write the old buffer or read the old x)."""
    import torch

    from conftest import load_golden
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    u, ex = load_golden("ico2_helm_compress")
    dop = DeviceOperator(pack(u), device="cuda:0")
    rng = np.random.default_rng(3)
    pairs = []
    for _ in range(2):
        xs = {a: torch.empty(len(ex["vf_0" if not a else "va_0"]), dtype=torch.complex128).pin_memory() for a in (False, True)}
        ws = {a: torch.empty(len(ex["ref_fwd_0" if not a else "ref_adj_0"]), dtype=torch.complex128).pin_memory() for a in (False, True)}
        pairs.append((xs, ws))
    for step in range(40):
        adjoint = bool(rng.integers(2))
        vk, rk = ("va_0", "ref_adj_0") if adjoint else ("vf_0", "ref_fwd_0")
        s = complex(rng.standard_normal(), rng.standard_normal())
        which = int(rng.integers(3))
        host_io = [None, True, False][int(rng.integers(3))]
        if which < 2:
            xs, ws = pairs[which]
            xs[adjoint].numpy()[:] = np.asarray(ex[vk]) * s
            ws[adjoint].numpy()[:] = np.nan
            w = dop.matvec_host(xs[adjoint].numpy(), adjoint=adjoint, out=ws[adjoint].numpy(), host_io=host_io)
        else:
            w = dop.matvec_host(np.asarray(ex[vk]) * s, adjoint=adjoint, host_io=host_io)
        assert rel(w, np.asarray(ex[rk]) * s) <= 1e-12, (step, adjoint, which, host_io)


def test_matmat_host_pipelined():
    """uhmv_matmat_host: host X in 16-column chunks, H2D / DMMA / D2H overlapped on three
    streams -- every column vs the reference's column loop (oracle), fwd + adj, 1e-12."""
    import torch

    from conftest import load_golden
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    u, ex = load_golden("helm400")
    dop = DeviceOperator(pack(u), device="cuda:0")
    rng = np.random.default_rng(11)
    for adjoint in (False, True):
        n_in = u.shape[0] if adjoint else u.shape[1]
        X = torch.from_numpy(rng.standard_normal((n_in, 48)) + 1j * rng.standard_normal((n_in, 48))).pin_memory()
        W = dop.matmat_host(X.numpy(), adjoint=adjoint, chunk=16)
        for j in (0, 17, 47):
            assert rel(W[:, j], oracle_matvec_uh(u, X.numpy()[:, j], adjoint=adjoint)) <= TOL, (adjoint, j)
        W2 = dop.matmat(X.cuda(), adjoint=adjoint).cpu().numpy()
        assert rel(W, W2) <= 1e-14
