"""Multi-GPU uniform-H matvec: row-cluster partition + one y/u all-gather.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank r owns a
contiguous slice of output leaves (``packer.partition_bounds``) and the input clusters whose
first index falls in its input slice.  A matvec on every rank is

    launch A   P1 / RED / U for owned input clusters (+ nearfield of its rows)   -> y, u
    exchange   in-place all-gather of the y/u exchange region (per-rank blocks, padded)
    launch B   Z for output clusters touching its rows, FAR (+ rest of nearfield) -> w[rows]

so the only data-path communication is the small coefficient exchange (~1 MB at config 3,
vs 2.6 GB of operator).

``exchange="peer"`` fuses the exchange into the kernel instead: ONE launch per rank
(``pack(peer=True)``) whose P1 / RED / U ops store this rank's y_t / u_t straight into every
rank's work buffer over the NVLink peer mappings (torch symmetric memory) and signal the
peers' dependency counters with system-scope releases; the Z ops wait on those counters, so
the transfer overlaps the nearfield and the rest of the farfield op by op
(csrc/uhmv_bulk.cuh, PEER).  ``PeerEmulation`` runs the same programs for all ranks in one
launch on one GPU (each rank on its share of the SMs, peers' buffers on the same device) --
the way the protocol is verified and measured with one GPU.  x is replicated; each rank's w holds its own rows (``gather=True``
all-gathers the full vector).  This replaces the reference's implicit hand-off of the
``stage`` dict across its thread-pool join (uniform.py:507, :518, :535).
"""

from __future__ import annotations

import numpy as np

from .packer import pack

__all__ = ["DistributedOperator", "PeerEmulation", "exchange_views", "make_distributed"]


def exchange_views(work, packed, adjoint: bool):
    """(region, mine): the y/u exchange region of a work tensor and this rank's block."""
    off, ex_len = packed.exchange["adj" if adjoint else "fwd"]
    world, rank = packed.world, packed.rank
    region = work[off : off + world * ex_len]
    mine = region[rank * ex_len : (rank + 1) * ex_len]
    return region, mine


def _check_vec(t, n, device, name):
    """C-ABI buffers are raw pointers: a wrong size, dtype, stride or device is refused here."""
    import torch

    if (not isinstance(t, torch.Tensor) or t.dtype != torch.complex128 or t.device != device
            or tuple(t.shape) != (n,) or not t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous complex128 {device} tensor of shape ({n},)")


def _peer_rank(work, work_len, counters, done):
    from . import _lib

    r = _lib.UhmvPeerRank()
    r.work, r.work_len, r.counters, r.done = int(work), int(work_len), int(counters), int(done)
    return r


def _execute_peer(plans, rank0, world, ranks, x, ws, adjoint, epoch, stream):
    import ctypes

    from . import _lib

    n = len(plans)
    rc = _lib.lib().uhmv_execute_peer(
        (ctypes.c_void_p * n)(*[p.value for p in plans]), n, rank0, world,
        (_lib.UhmvPeerRank * world)(*ranks), ctypes.c_void_p(x.data_ptr()),
        (ctypes.c_void_p * n)(*[w.data_ptr() for w in ws]), int(adjoint), ctypes.c_uint32(epoch),
        ctypes.c_void_p(stream.cuda_stream),
    )
    _lib.check(rc, "uhmv_execute_peer")


class PeerEmulation:
    """Every rank of a peer-exchange partition in ONE launch on one GPU.

    Rank r's CTAs run its own program (``pack(u, rank=r, world=world, peer=True)``) on 1/world
    of the SMs, with its own work / counter / done buffers; the "peer" pointers are the other
    ranks' buffers on the same device.  Ranks wait on one another inside the one launch (all
    CTAs are co-resident), never across launches.  All ranks add their disjoint rows into one
    output vector, so ``matvec`` returns the full product."""

    def __init__(self, u, world: int, device=None, packs=None):
        import torch

        from .device import DeviceOperator

        if not 1 <= world <= 8:
            raise ValueError("peer partitions span 1..8 ranks (one NVLink domain)")
        self.world = world
        if packs is None:
            base = pack(u, rank=0, world=world, peer=True)
            packs = [base] + [base.for_rank(r, world, peer=True) for r in range(1, world)]
        self.packs = packs
        # every rank reads the same arena: one copy, padded for the widest TMA leading dimension
        def pad(p):
            return max([int(q.mr_lds.max()) for q in (p.fwd, p.adj) if q.mr_lds is not None and len(q.mr_lds)] + [0])

        first = max(range(world), key=lambda r: pad(self.packs[r]))
        owner = DeviceOperator(self.packs[first], device=device)
        self.ops = [owner if r == first else DeviceOperator(p, device=device, share_arena_with=owner)
                    for r, p in enumerate(self.packs)]
        self.device = self.ops[0].device
        p0 = self.packs[0]
        self.n_rows, self.n_cols = p0.n_rows, p0.n_cols
        # per direction (forward / adjoint have their own counter numbering and epochs): every
        # rank's work buffer (two epoch halves), dependency counters and done-epoch flags
        n_ctr = [max(p.fwd.n_counters, p.adj.n_counters, 1) for p in self.packs]
        self._bufs = []
        self.ranks = {}
        for adjoint in (False, True):
            bufs = [(torch.zeros(2 * max(p.work_len, 1), dtype=torch.complex128, device=self.device),
                     torch.zeros(n, dtype=torch.int32, device=self.device),
                     torch.zeros(world, dtype=torch.int32, device=self.device)) for p, n in zip(self.packs, n_ctr)]
            self._bufs.append(bufs)
            self.ranks[adjoint] = [_peer_rank(w.data_ptr(), max(p.work_len, 1), c.data_ptr(), d.data_ptr())
                                   for (w, c, d), p in zip(bufs, self.packs)]
        self.epoch = {False: 0, True: 0}

    @property
    def arena_bytes(self) -> int:
        return 16 * sum(p.fwd.arena_elems for p in self.packs)

    def kernel_launches(self, adjoint=False, mode=None) -> int:
        return 1

    def launch_info(self, adjoint=False, mode=None):
        info = self.ops[0].launch_info(adjoint, "bulk")
        info["ranks"] = self.world
        return info

    def matvec_host(self, x_host, adjoint=False, out=None, mode=None):
        """Host buffers: H2D of x, the one launch, D2H of w, synchronize."""
        torch = self.ops[0].torch
        x = torch.from_numpy(np.ascontiguousarray(x_host, dtype=np.complex128)).to(self.device, non_blocking=True)
        w = self.matvec(x, adjoint=adjoint).cpu().numpy()
        if out is not None:
            out[...] = w
            return out
        return w

    def matvec(self, x, adjoint=False, out=None, stream=None, mode=None):
        torch = self.ops[0].torch
        n_in, n_out = (self.n_rows, self.n_cols) if adjoint else (self.n_cols, self.n_rows)
        if x.shape != (n_in,) or x.dtype != torch.complex128 or x.device != self.device:
            raise ValueError(f"x must be a complex128 {self.device} tensor of shape ({n_in},)")
        x = x.contiguous()
        if out is None:
            out = torch.empty(n_out, dtype=torch.complex128, device=self.device)
        _check_vec(out, n_out, self.device, "out")
        adjoint = bool(adjoint)
        self.epoch[adjoint] += 1
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _execute_peer([op._plan for op in self.ops], 0, self.world, self.ranks[adjoint], x, [out] * self.world,
                      adjoint, self.epoch[adjoint], st)
        return out


class DistributedOperator:
    """This rank's share of a packed operator, resident on its GPU.

    ``exchange="nccl"`` (default): launch A, in-place NCCL all-gather of y/u, launch B.
    ``exchange="peer"``: one launch per rank, y/u stored into the peers' work buffers inside
    the kernel (NVLink peer mappings from torch symmetric memory)."""

    def __init__(self, u, rank: int, world: int, device=None, group=None, exchange: str = "nccl", packed=None):
        from .device import DeviceOperator

        if exchange not in ("nccl", "peer"):
            raise ValueError("exchange is 'nccl' or 'peer'")
        self.rank, self.world, self.group, self.exchange = rank, world, group, exchange
        if packed is None:
            packed = pack(u, rank=rank, world=world, peer=exchange == "peer")
        self.packed_local = packed
        self.a = DeviceOperator(packed, device=device)
        if exchange == "peer":
            self.b = None
            self._setup_peer()
        elif packed.fwd.part_b is None:  # world 1: nothing to exchange
            self.b = None
        else:
            self.b = DeviceOperator(
                packed, device=device, programs=(packed.fwd.part_b, packed.adj.part_b), share_with=self.a
            )
        self.device = self.a.device
        self.n_rows, self.n_cols = packed.n_rows, packed.n_cols
        part = packed.part
        if part is None:  # world 1
            self.row_slice, self.col_slice = (0, self.n_rows), (0, self.n_cols)
        else:
            self.row_slice = (part["row_bounds"][rank], part["row_bounds"][rank + 1])
            self.col_slice = (part["col_bounds"][rank], part["col_bounds"][rank + 1])

    def _setup_peer(self):
        """One symmetric-memory allocation per rank holds its peer-visible buffers: work (two
        epoch halves), dependency counters, done-epoch flags; every rank maps every other's."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        p = self.packed_local
        dev = self.a.device
        meta = torch.tensor([max(p.work_len, 1), max(p.fwd.n_counters, p.adj.n_counters, 1)], dtype=torch.int64,
                            device=dev)
        lens = [torch.zeros_like(meta) for _ in range(self.world)]
        dist.all_gather(lens, meta, group=self.group)
        work_lens = [int(t[0]) for t in lens]
        wmax, cmax = max(work_lens), max(int(t[1]) for t in lens)
        off_c = 2 * wmax * 16
        off_d = off_c + ((4 * cmax + 127) // 128) * 128
        per_dir = off_d + ((4 * self.world + 127) // 128) * 128  # forward block, then adjoint block
        # every rank must reach the (collective) rendezvous or none: agree on the allocation first
        try:
            self._symm_buf = symm.empty(2 * per_dir, dtype=torch.uint8, device=dev)
            self._symm_buf.zero_()
            ok = 1
        except Exception:  # noqa: BLE001
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        if int(flag.item()) == 0:
            raise RuntimeError("symmetric-memory allocation failed on some rank")
        torch.cuda.synchronize(dev)
        grp = self.group if self.group is not None else dist.group.WORLD
        try:
            self._symm = symm.rendezvous(self._symm_buf, grp.group_name)
        except RuntimeError:  # older releases: symmetric memory is enabled per group first
            symm.enable_symm_mem_for_group(grp.group_name)
            self._symm = symm.rendezvous(self._symm_buf, grp.group_name)
        ptrs = list(self._symm.buffer_ptrs)
        self.ranks = {
            adjoint: [_peer_rank(ptrs[q] + b, work_lens[q], ptrs[q] + b + off_c, ptrs[q] + b + off_d)
                      for q in range(self.world)]
            for adjoint, b in ((False, 0), (True, per_dir))
        }
        self.epoch = {False: 0, True: 0}
        dist.barrier(group=self.group)

    @property
    def arena_bytes(self) -> int:
        """Operator bytes this rank streams per forward matvec (roofline numerator)."""
        p = self.packed_local
        if self.exchange == "peer":
            return 16 * p.fwd.arena_elems
        return 16 * (p.fwd.arena_elems + p.fwd.part_b.arena_elems)

    def kernel_launches(self, adjoint=False, mode=None) -> int:
        if self.exchange == "peer":
            return 1
        return self.a.kernel_launches(adjoint, mode) + (self.b.kernel_launches(adjoint, mode) if self.b else 0)

    def launch_info(self, adjoint=False, mode=None):
        return self.a.launch_info(adjoint, mode)

    def matvec(self, x, adjoint=False, out=None, mode=None, gather=False):
        if self.exchange == "peer":
            torch = self.a.torch
            n_in, n_out = (self.n_rows, self.n_cols) if adjoint else (self.n_cols, self.n_rows)
            _check_vec(x, n_in, self.device, "x")
            if out is None:
                out = torch.empty(n_out, dtype=torch.complex128, device=self.device)
            _check_vec(out, n_out, self.device, "out")
            adjoint = bool(adjoint)
            self.epoch[adjoint] += 1
            _execute_peer([self.a._plan], self.rank, self.world, self.ranks[adjoint], x.contiguous(), [out], adjoint,
                          self.epoch[adjoint], torch.cuda.current_stream(self.device))
            return self.gather_output(out, adjoint) if gather else out
        out = self.a.matvec(x, adjoint=adjoint, out=out, mode=mode)
        if self.b is None:  # world 1
            return out
        region, mine = exchange_views(self.a.work, self.packed_local, adjoint)
        if region.numel():
            self._all_gather(region, mine)
        out = self.b.matvec(x, adjoint=adjoint, out=out, mode=mode)
        if gather:
            out = self.gather_output(out, adjoint)
        return out

    def _all_gather(self, out, inp):
        """all_gather_into_tensor over the group; NCCL works on the device buffers in place.
        A gloo group (multi-process tests on one GPU) stages through host memory."""
        import torch
        import torch.distributed as dist

        if out.is_cuda and dist.get_backend(self.group) == "gloo":
            host = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather_into_tensor(torch.view_as_real(host), torch.view_as_real(inp.cpu()), group=self.group)
            out.copy_(host)
            return
        dist.all_gather_into_tensor(torch.view_as_real(out), torch.view_as_real(inp), group=self.group)

    def gather_output(self, w, adjoint=False):
        """All-gather the ranks' output slices into the full vector (padded blocks)."""
        import torch

        if self.world == 1:
            return w
        bounds = self.packed_local.part["col_bounds" if adjoint else "row_bounds"]
        lens = np.diff(bounds)
        blk = int(lens.max())
        lo, hi = bounds[self.rank], bounds[self.rank + 1]
        send = torch.zeros(blk, dtype=w.dtype, device=w.device)
        send[: hi - lo] = w[lo:hi]
        recv = torch.empty(blk * self.world, dtype=w.dtype, device=w.device)
        self._all_gather(recv, send)
        full = torch.empty_like(w)
        for r in range(self.world):
            full[bounds[r] : bounds[r + 1]] = recv[r * blk : r * blk + lens[r]]
        return full

    def matvec_host(self, x_host, adjoint=False, out=None, mode=None):
        import torch

        x = torch.from_numpy(np.ascontiguousarray(x_host, dtype=np.complex128)).to(self.device)
        w = self.matvec(x, adjoint=adjoint, mode=mode, gather=True).cpu().numpy()
        if out is not None:
            out[...] = w
            return out
        return w


def make_distributed(u, rank: int, world: int, device=None, group=None, exchange: str = "auto", check_tol=1e-12):
    """The rank's DistributedOperator.  ``exchange="auto"``: the fused peer exchange when every
    rank can map every other's buffers (torch symmetric memory) AND its first forward and
    adjoint matvecs on a seeded vector agree with the NCCL path within ``check_tol`` on every
    rank; the NCCL path otherwise.  Returns (operator, reason)."""
    import torch
    import torch.distributed as dist

    if exchange in ("nccl", "peer"):
        return DistributedOperator(u, rank, world, device=device, group=group, exchange=exchange), "requested"
    base = pack(u, rank=rank, world=world, peer=True)
    nccl = DistributedOperator(u, rank, world, device=device, group=group, exchange="nccl",
                               packed=base.for_rank(rank, world, peer=False))
    dev = nccl.device
    peer, why = None, ""
    try:
        peer = DistributedOperator(u, rank, world, device=device, group=group, exchange="peer", packed=base)
        ok = 1
    except Exception as e:  # noqa: BLE001 -- any rank unable to map its peers: NCCL everywhere
        ok, why = 0, f"peer setup failed: {type(e).__name__}: {e}"[:200]
    flag = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 1:
        g = torch.Generator(device="cpu").manual_seed(1234)
        err = 0.0
        for adjoint in (False, True):
            n_in = u.shape[0] if adjoint else u.shape[1]
            x = torch.complex(torch.randn(n_in, generator=g, dtype=torch.float64),
                              torch.randn(n_in, generator=g, dtype=torch.float64)).to(dev)
            a = nccl.matvec(x, adjoint=adjoint, gather=True)
            b = peer.matvec(x, adjoint=adjoint, gather=True)
            err = max(err, float(torch.linalg.norm(a - b) / torch.linalg.norm(a)))
        e = torch.tensor([err], dtype=torch.float64, device=dev)
        dist.all_reduce(e, op=dist.ReduceOp.MAX, group=group)
        if float(e.item()) <= check_tol:
            del nccl
            return peer, f"peer exchange (agrees with the NCCL path to {float(e.item()):.1e})"
        why = f"peer result differs from the NCCL path ({float(e.item()):.1e})"
    elif not why:
        why = "a peer rank could not map its buffers"
    del peer
    return nccl, "NCCL all-gather: " + why
