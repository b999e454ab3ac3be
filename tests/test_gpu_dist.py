"""Partitioned matvec on the device engine: world_size 2 and 3, every rank a real process.

Each rank builds ``dist.DistributedOperator`` (its launch-A / launch-B programs resident on
cuda:0), runs the two CUDA launches around the y/u exchange and all-gathers its output
slice.  The round's GPU pool gives one GPU per call, so the ranks share cuda:0 and exchange
over gloo (staged through host memory); the kernels of different ranks never wait on each
other -- the only cross-rank dependency is the collective between launch A and launch B,
exactly as under NCCL.  Checked against the reference's stored outputs at 1e-12."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, mode, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_15573_b200.dist import DistributedOperator
        from paper_2405_15573_b200.uh_io import load_uh

        u, ex = load_uh(os.path.join(GOLDEN, f"{name}.npz"))
        dev = torch.device("cuda", 0)
        op = DistributedOperator(u, rank, world, device=dev)
        errs = {}
        for adjoint, vkey, rkey in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
            x = torch.from_numpy(np.asarray(ex[vkey], dtype=np.complex128)).to(dev)
            for rep in range(2):  # second call: counters self-reset, w re-zeroed
                w = op.matvec(x, adjoint=adjoint, mode=mode, gather=True).cpu().numpy()
            ref = ex[rkey]
            errs[adjoint] = float(np.linalg.norm(w - ref) / np.linalg.norm(ref))
            wh = op.matvec_host(ex[vkey], adjoint=adjoint, mode=mode)
            errs[f"host{int(adjoint)}"] = float(np.linalg.norm(wh - ref) / np.linalg.norm(ref))
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["bulk", "fused"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["helm400", "ico2_helm_compress", "rect_sphere"])
def test_partitioned_matvec_device(name, world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, mode, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    for _ in range(world):
        rank, errs = q.get(timeout=5)
        assert all(v <= 1e-12 for v in errs.values()), (rank, errs)
