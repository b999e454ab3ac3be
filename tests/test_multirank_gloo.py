"""Multi-rank (row-cluster partition) logic on CPU: world_size 2 and 3 over gloo.

Each rank packs its share (packer.pack(rank=, world=)), runs launch A with the NumPy VM
(oracle/packed_vm.py: the device program semantics), exchanges the y/u region with a real
torch.distributed all_gather_into_tensor (gloo), runs launch B, and the ranks' output
slices are gathered and checked against the reference's stored outputs (1e-12)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from packed_vm import run_program
        from paper_2405_15573_b200.packer import pack, partition_bounds
        from paper_2405_15573_b200.uh_io import load_uh

        u, ex = load_uh(os.path.join(GOLDEN, f"{name}.npz"))
        p = pack(u, rank=rank, world=world)
        errs = {}
        for adjoint, vkey, rkey, fkey in ((False, "vf_0", "ref_fwd_0", "ref_far_fwd_0"), (True, "va_0", "ref_adj_0", "ref_far_adj_0")):
            prog = p.adj if adjoint else p.fwd
            x = np.asarray(ex[vkey], dtype=np.complex128)
            n_out = p.n_cols if adjoint else p.n_rows
            w = np.zeros(n_out, dtype=np.complex128)
            work = np.zeros(p.work_len, dtype=np.complex128)
            run_program(prog, p.arena, work, x, w, order="fused", engine="pieces")
            off, ex_len = p.exchange["adj" if adjoint else "fwd"]
            region = torch.from_numpy(work[off : off + world * ex_len])
            mine = region[rank * ex_len : (rank + 1) * ex_len].clone()
            if region.numel():
                dist.all_gather_into_tensor(torch.view_as_real(region), torch.view_as_real(mine))
            run_program(prog.part_b, p.arena, work, x, w, order="fused", engine="pieces")
            bounds = p.part["col_bounds" if adjoint else "row_bounds"]
            lo, hi = bounds[rank], bounds[rank + 1]
            # rows outside the slice stay untouched (zero)
            outside = np.concatenate([w[:lo], w[hi:]])
            assert not outside.any()
            parts = [None] * world
            dist.all_gather_object(parts, (lo, hi, w[lo:hi]))
            full = np.zeros(n_out, dtype=np.complex128)
            for a, b, piece in parts:
                full[a:b] = piece
            ref = ex[rkey]
            errs[adjoint] = float(np.linalg.norm(full - ref) / np.linalg.norm(ref))
            # each rank streams a share of the operator; shares add up to the whole
            share = torch.tensor([prog.arena_elems + prog.part_b.arena_elems], dtype=torch.float64)
            dist.all_reduce(share)
            errs[f"share{int(adjoint)}"] = float(share.item())
        if rank == 0:
            q.put((errs, (p.fwd.arena_elems, p.bytes_alg // 16)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["ico2_helm_compress", "uh800_laplace", "rect_sphere"])
def test_partitioned_matvec_gloo(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    errs, _ = q.get(timeout=5)
    assert errs[False] <= 1e-12 and errs[True] <= 1e-12, errs
    from conftest import load_golden
    from paper_2405_15573_b200.packer import pack

    u, _ = load_golden(name)
    total = pack(u).bytes_alg // 16
    # every operator element is streamed by exactly one rank (Z of output clusters that
    # straddle a cut would be duplicated; none at these sizes is allowed to exceed 10%)
    assert total <= errs["share0"] <= 1.1 * total


def test_partition_bounds_cover():
    from conftest import load_golden
    from paper_2405_15573_b200.packer import partition_bounds

    u, _ = load_golden("uh800_laplace")
    for world in (1, 2, 3, 4, 8):
        b = partition_bounds(u.bct.row_tree, world)
        assert b[0] == 0 and b[-1] == 800 and all(x < y for x, y in zip(b, b[1:]))
        leaf_ends = {n.hi for n in u.bct.row_tree.nodes if n.is_leaf} | {0}
        assert set(b) <= leaf_ends


def _peer_worker(rank, world, port, name, shm_names, shapes, q):
    """One rank of the peer-exchange protocol in its own process: work / counters / done of
    every rank live in shared memory (the CPU stand-in for the NVLink peer mappings)."""
    import random
    import sys
    from multiprocessing import shared_memory

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shms = []
    try:
        from packed_vm import run_peer_rank
        from paper_2405_15573_b200.packer import pack
        from paper_2405_15573_b200.uh_io import load_uh

        u, ex = load_uh(os.path.join(GOLDEN, f"{name}.npz"))
        p = pack(u, rank=rank, world=world, peer=True)

        def view(nm, shape, dtype):
            s = shared_memory.SharedMemory(name=nm)
            shms.append(s)
            return np.ndarray(shape, dtype=dtype, buffer=s.buf)

        errs = {}
        for adjoint, vkey, rkey in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
            d = "adj" if adjoint else "fwd"
            work = [view(shm_names[d]["work"][r], shapes[d]["work"][r], np.complex128) for r in range(world)]
            ctrs = [view(shm_names[d]["ctr"][r], shapes[d]["ctr"][r], np.int64) for r in range(world)]
            done = [view(shm_names[d]["done"][r], (world,), np.int64) for r in range(world)]
            lock = q[1]
            x = np.asarray(ex[vkey], dtype=np.complex128)
            n_out = p.n_cols if adjoint else p.n_rows
            w = np.zeros(n_out, dtype=np.complex128)
            dist.barrier()

            def scale(e):  # a different x every epoch: stale exchange data would show
                return 1.0 + 0.37j * e

            rng = random.Random(rank * 7 + int(adjoint))

            class Jitter:  # rank 0 races ahead, the others lag
                def random(self):
                    return rng.random() * (0.05 if rank == 0 else 3.0)

            outs = run_peer_rank(p, rank, world, work, ctrs, done, x, w, adjoint=adjoint, epochs=5, lock=lock,
                                 jitter=Jitter(), scale=scale)
            parts = [None] * world
            dist.all_gather_object(parts, outs)
            ref = ex[rkey]
            e_max = 0.0
            for e in range(len(outs)):
                full = np.sum([pt[e] for pt in parts], axis=0)  # ranks own disjoint rows
                refe = ref * scale(e + 1)
                e_max = max(e_max, float(np.linalg.norm(full - refe) / np.linalg.norm(refe)))
            errs[adjoint] = e_max
        if rank == 0:
            q[0].put(errs)
    finally:
        for s in shms:
            s.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["ico2_helm_compress", "rect_sphere"])
def test_peer_protocol_multiprocess_gloo(name, world):
    """The peer-exchange protocol with REAL concurrency: world processes (gloo rendezvous),
    each running its rank's program over shared-memory peer buffers, 5 consecutive epochs per
    direction with a different x each (monotonic counters, two work halves, done-epoch guard),
    rank 0 racing ahead of the others; every epoch's gathered output matches the reference
    (linearity: x * s_e -> ref * s_e) at 1e-12.  Satisfying a wait one arrival early makes it
    fail (stale or missing exchange data).  (The done-epoch guard is a safety net for ranks
    that consume nothing from some peer; on these operators every rank consumes from every
    other, which already keeps them within one epoch of each other.)"""
    from multiprocessing import shared_memory

    from conftest import load_golden
    from paper_2405_15573_b200.packer import pack

    u, _ = load_golden(name)
    ctx = mp.get_context("spawn")
    packs = [pack(u, rank=r, world=world, peer=True) for r in range(world)]
    shms, names, shapes = [], {}, {}
    for d in ("fwd", "adj"):
        names[d], shapes[d] = {"work": [], "ctr": [], "done": []}, {"work": [], "ctr": []}
        for p in packs:
            prog = p.adj if d == "adj" else p.fwd
            for key, shape, dt in (("work", (2, max(p.work_len, 1)), np.complex128),
                                   ("ctr", (max(prog.n_counters, 1),), np.int64), ("done", (world,), np.int64)):
                s = shared_memory.SharedMemory(create=True, size=int(np.prod(shape)) * np.dtype(dt).itemsize)
                np.ndarray(shape, dtype=dt, buffer=s.buf)[...] = 0
                shms.append(s)
                names[d][key].append(s.name)
                if key != "done":
                    shapes[d][key].append(shape)
    try:
        q = (ctx.Queue(), ctx.Lock())
        port = _free_port()
        procs = [ctx.Process(target=_peer_worker, args=(r, world, port, name, names, shapes, q)) for r in range(world)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(timeout=600)
        assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
        errs = q[0].get(timeout=5)
        assert errs[False] <= 1e-12 and errs[True] <= 1e-12, errs
    finally:
        for s in shms:
            s.close()
            s.unlink()
