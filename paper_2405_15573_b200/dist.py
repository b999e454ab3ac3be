"""Multi-GPU uniform-H matvec: row-cluster partition + one y/u all-gather.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank r owns a
contiguous slice of output leaves (``packer.partition_bounds``) and the input clusters whose
first index falls in its input slice.  A matvec on every rank is

    launch A   P1 / RED / U for owned input clusters (+ nearfield of its rows)   -> y, u
    exchange   in-place all-gather of the y/u exchange region (per-rank blocks, padded)
    launch B   Z for output clusters touching its rows, FAR (+ rest of nearfield) -> w[rows]

so the only data-path communication is the small coefficient exchange (~1 MB at config 3,
vs 2.6 GB of operator).  x is replicated; each rank's w holds its own rows (``gather=True``
all-gathers the full vector).  This replaces the reference's implicit hand-off of the
``stage`` dict across its thread-pool join (uniform.py:507, :518, :535).
"""

from __future__ import annotations

import numpy as np

from .packer import pack

__all__ = ["DistributedOperator", "exchange_views"]


def exchange_views(work, packed, adjoint: bool):
    """(region, mine): the y/u exchange region of a work tensor and this rank's block."""
    off, ex_len = packed.exchange["adj" if adjoint else "fwd"]
    world, rank = packed.world, packed.rank
    region = work[off : off + world * ex_len]
    mine = region[rank * ex_len : (rank + 1) * ex_len]
    return region, mine


class DistributedOperator:
    """This rank's share of a packed operator, resident on its GPU."""

    def __init__(self, u, rank: int, world: int, device=None, group=None):
        from .device import DeviceOperator

        self.rank, self.world, self.group = rank, world, group
        self.packed_local = packed = pack(u, rank=rank, world=world)
        self.a = DeviceOperator(packed, device=device)
        self.b = DeviceOperator(
            packed, device=device, programs=(packed.fwd.part_b, packed.adj.part_b), share_with=self.a
        )
        self.device = self.a.device
        self.n_rows, self.n_cols = packed.n_rows, packed.n_cols
        part = packed.part
        self.row_slice = (part["row_bounds"][rank], part["row_bounds"][rank + 1])
        self.col_slice = (part["col_bounds"][rank], part["col_bounds"][rank + 1])

    @property
    def arena_bytes(self) -> int:
        """Operator bytes this rank streams per forward matvec (roofline numerator)."""
        p = self.packed_local
        return 16 * (p.fwd.arena_elems + p.fwd.part_b.arena_elems)

    def kernel_launches(self, adjoint=False, mode=None) -> int:
        return self.a.kernel_launches(adjoint, mode) + self.b.kernel_launches(adjoint, mode)

    def launch_info(self, adjoint=False, mode=None):
        return self.a.launch_info(adjoint, mode)

    def matvec(self, x, adjoint=False, out=None, mode=None, gather=False):
        out = self.a.matvec(x, adjoint=adjoint, out=out, mode=mode)
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
