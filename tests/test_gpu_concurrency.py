"""One plan shared by several streams and host threads (include/uhmv.h "Concurrency").

A plan's launches own its ticket / counters / work buffer, and the multi-RHS plan shares them
(device.py share_with): the C layer serialises every launch of such a group (group mutex +
event).  Interleaving matvec and matmat calls on two streams -- and from two host threads --
must give the bit-identical results of the serial calls."""

import threading

import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _setup(name="helm400"):
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    u, ex = load_golden(name)
    dop = DeviceOperator(pack(u), device="cuda:0")
    n = u.shape[1]
    rng = np.random.default_rng(11)
    xs = [torch.from_numpy(rng.standard_normal(n) + 1j * rng.standard_normal(n)).to("cuda:0") for _ in range(8)]
    X = torch.from_numpy(rng.standard_normal((n, 16)) + 1j * rng.standard_normal((n, 16))).to("cuda:0")
    return dop, xs, X


def test_two_streams_interleaved_bitwise():
    dop, xs, X = _setup()
    serial = [dop.matvec(x, adjoint=(i % 2 == 1)).clone() for i, x in enumerate(xs)]
    serial_mm = dop.matmat(X).clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs, mms = [], []
    for it in range(50):
        st = s1 if it % 2 == 0 else s2
        with torch.cuda.stream(st):
            i = it % len(xs)
            outs.append((i, dop.matvec(xs[i], adjoint=(i % 2 == 1))))
            if it % 5 == 0:
                mms.append(dop.matmat(X))
    torch.cuda.synchronize()
    for i, w in outs:
        assert torch.equal(w, serial[i]), i
    for W in mms:
        assert torch.equal(W, serial_mm)


def test_two_host_threads_bitwise():
    dop, xs, X = _setup()
    serial = [dop.matvec(x).clone() for x in xs]
    torch.cuda.synchronize()
    errors = []

    def worker(seed):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for it in range(50):
                    i = (it + seed) % len(xs)
                    w = dop.matvec(xs[i])
                    st.synchronize()
                    if not torch.equal(w, serial[i]):
                        errors.append((seed, it))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:5]


def test_host_calls_two_threads_bitwise():
    """uhmv_matvec_host shares the plan's scratch vectors and graphs across threads."""
    dop, xs, _ = _setup()
    xh = [x.cpu().numpy() for x in xs]
    serial = [dop.matvec_host(x) for x in xh]
    errors = []

    def worker(seed):
        for it in range(30):
            i = (it + seed) % len(xh)
            w = dop.matvec_host(xh[i])
            if not np.array_equal(w, serial[i]):
                errors.append((seed, it))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:5]


def test_out_buffer_validation():
    dop, xs, X = _setup()
    n = xs[0].shape[0]
    with pytest.raises(ValueError):
        dop.matvec(xs[0], out=torch.empty(n - 1, dtype=torch.complex128, device="cuda:0"))
    with pytest.raises(ValueError):
        dop.matvec(xs[0], out=torch.empty(2 * n, dtype=torch.complex128, device="cuda:0")[::2])
    with pytest.raises(ValueError):
        dop.matvec(xs[0], out=torch.empty(n, dtype=torch.complex64, device="cuda:0"))
    with pytest.raises(ValueError):
        dop.matvec(xs[0], out=torch.empty(n, dtype=torch.complex128))
    with pytest.raises(ValueError):
        dop.matmat(X.cpu())
