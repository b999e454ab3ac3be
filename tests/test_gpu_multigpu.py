"""Real multi-GPU runs (one process per GPU, NCCL): skipped unless >= 2 GPUs are visible.

The round's GPU pool gives one GPU per call, so this runs whenever a multi-GPU box is used:
it exercises what a single GPU cannot -- the NCCL all-gather between launch A and B, and the
fused peer exchange's cross-device memory ordering over NVLink (st / red / ld at .sys scope,
csrc/uhmv_bulk.cuh PEER) -- for W = 2 and all visible GPUs, forward and adjoint, 20 epochs
per direction with distinct vectors, against the CPU oracle at 1e-12 and against the NCCL path
at 1e-14."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import GOLDEN, ROOT

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs"),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q):
    import sys

    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from matvec_oracle import oracle_matvec_uh

        from paper_2405_15573_b200 import workloads
        from paper_2405_15573_b200.dist import DistributedOperator
        from paper_2405_15573_b200.uh_io import load_uh

        u = workloads.build_operator(2) if name == "cfg2" else load_uh(os.path.join(GOLDEN, f"{name}.npz"))[0]
        ops = {ex: DistributedOperator(u, rank, world, device=dev, exchange=ex) for ex in ("nccl", "peer")}
        worst, same = 0.0, True
        for epoch in range(20):
            for adjoint in (False, True):
                n_in = u.shape[0] if adjoint else u.shape[1]
                rng = np.random.default_rng(100 * epoch + adjoint)
                v = rng.standard_normal(n_in) + 1j * rng.standard_normal(n_in)
                x = torch.from_numpy(v).to(dev)
                a = ops["nccl"].matvec(x, adjoint=adjoint, gather=True).cpu().numpy()
                b = ops["peer"].matvec(x, adjoint=adjoint, gather=True).cpu().numpy()
                same = same and float(np.linalg.norm(a - b) / np.linalg.norm(a)) <= 1e-14
                if epoch % 5 == 0:
                    ref = oracle_matvec_uh(u, v, adjoint=adjoint)
                    worst = max(worst, float(np.linalg.norm(b - ref) / np.linalg.norm(ref)))
        q.put((rank, worst, same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["helm400", "ico2_helm_compress", "cfg2"])
@pytest.mark.parametrize("world", sorted({2, min(torch.cuda.device_count(), 8)} if torch.cuda.is_available() else {2}))
def test_multi_gpu_nccl_and_peer(name, world):
    import torch.multiprocessing as mp

    if world < 2:
        pytest.skip("needs >= 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=900)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    for _ in range(world):
        rank, worst, same = q.get(timeout=5)
        assert worst <= 1e-12 and same, (rank, worst, same)
