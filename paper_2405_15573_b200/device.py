"""Device-resident packed operator: PyTorch owns the buffers, libuhmv.so runs the kernels.

PyTorch is plumbing here (device memory, streams, torch.distributed); every FLOP of the
matvec runs in the hand-written sm_100a kernels of csrc/uhmv.cu behind the C ABI of
include/uhmv.h.  There is no CPU or PyTorch fallback: without CUDA this raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time

import numpy as np

from . import _lib
from .packer import PackedOperator, Program

__all__ = ["DeviceOperator", "default_mode"]

_MODES = {"phased": _lib.MODE_PHASED, "fused": _lib.MODE_FUSED, "bulk": _lib.MODE_BULK}
MODES = tuple(_MODES)


def _torch_dtypes():
    import torch

    return {np.dtype(np.complex128): torch.complex128, np.dtype(np.complex64): torch.complex64,
            np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}


_TORCH_COPY_MIN = 65536  # complex elements (1 MB)
try:
    _TORCH_DTYPES = _torch_dtypes()
except ImportError:  # pragma: no cover
    _TORCH_DTYPES = {}


def default_mode() -> str:
    return os.environ.get("UHMV_MODE", "bulk")


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("uniform-H matvec needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch


class _DeviceProgram:
    def __init__(self, torch, prog: Program, device):
        def up(a, dtype):
            a = np.ascontiguousarray(a)
            if a.size == 0:
                a = np.zeros(1, dtype=a.dtype)
            return torch.from_numpy(a).to(device=device, dtype=dtype)

        self.prog = prog
        self.ops = up(prog.ops, torch.int32)
        self.segs = up(prog.segs, torch.int64)
        self.runs = up(prog.runs, torch.int64)
        self.waits = up(prog.waits, torch.int32)
        self.sigs = up(prog.sigs, torch.int32)
        self.fused_order = up(prog.fused_order, torch.int32)
        self.pieces = up(prog.pieces, torch.int64)
        self.mr_segs = up(prog.mr_segs, torch.int64)
        self.mr_ranges = up(prog.mr_ranges, torch.int32)
        # TMA tensor maps over the arena, one pair per leading dimension (filled by the plan)
        lds = prog.mr_lds if prog.mr_lds is not None else np.zeros(0, dtype=np.int64)
        self.tmap_lds = np.ascontiguousarray(lds, dtype=np.int64)
        self.tmaps = torch.zeros(max(1, 2 * len(lds)) * 128, dtype=torch.uint8, device=device)

    def struct(self) -> _lib.UhmvProgram:
        p = self.prog
        s = _lib.UhmvProgram()
        s.n_ops = p.n_ops
        s.ops = self.ops.data_ptr()
        s.segs = self.segs.data_ptr()
        s.runs = self.runs.data_ptr()
        s.waits = self.waits.data_ptr()
        s.sigs = self.sigs.data_ptr()
        s.fused_order = self.fused_order.data_ptr()
        s.pieces = self.pieces.data_ptr()
        if len(p.phases) > _lib.MAX_PHASES:
            raise ValueError("too many phases")
        s.n_phases = len(p.phases)
        for i, (a, b) in enumerate(p.phases):
            s.phase_lo[i] = a
            s.phase_hi[i] = b
        s.in_max = p.in_max
        s.out_max = p.out_max
        s.n_counters = p.n_counters
        s.xin_max = p.xin_max
        s.zero_output = int(p.zero_output)
        s.stage_elems = int(p.stage_elems)
        s.mr_segs = self.mr_segs.data_ptr()
        s.mr_ranges = self.mr_ranges.data_ptr()
        s.n_tmaps = len(self.tmap_lds)
        s.tmap_lds = self.tmap_lds.ctypes.data if len(self.tmap_lds) else None
        s.tmaps = self.tmaps.data_ptr()
        s.flags = (_lib.PROG_SYM if getattr(p, "bulk_only", False) else 0) | (_lib.PROG_XWIN if getattr(p, "xwin", False) else 0) | (
            _lib.PROG_WORDER if getattr(p, "w_order", False) else 0)
        return s


class DeviceOperator:
    """A packed uniform H-matrix resident in HBM, with its C-ABI plan."""

    def __init__(self, packed: PackedOperator, device=None, programs=None, share_with=None, share_arena_with=None,
                 guard: int = 0):
        """``programs=(fwd, adj)`` overrides the packed programs; ``share_with`` reuses another
        DeviceOperator's arena / work / counter buffers (multi-GPU launch B);
        ``share_arena_with`` reuses only its arena (the ranks of a peer-exchange emulation).
        ``guard`` > 0 (diagnostics, a compute-sanitizer stand-in): every buffer the kernels write
        gets ``guard`` sentinel elements on both sides; :meth:`check_guards` verifies them."""
        torch = _torch()
        L = _lib.lib()
        self.torch = torch
        self._guard = int(guard)
        self._guards = []
        self.packed = packed
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        fwd_p, adj_p = programs if programs is not None else (packed.fwd, packed.adj)
        self.progs = (fwd_p, adj_p)
        if share_with is not None:
            for name in ("arena", "work", "counters", "ticket", "exit_count", "x_scratch", "w_scratch"):
                setattr(self, name, getattr(share_with, name))
            lds = [int(q.mr_lds.max()) for q in (fwd_p, adj_p) if q.mr_lds is not None and len(q.mr_lds)]
            if max(lds + [0]) > share_with._arena_pad:
                raise ValueError("programs read the arena with a leading dimension beyond its padding")
            self._arena_pad = share_with._arena_pad
            need = max(fwd_p.n_counters, adj_p.n_counters, 1)
            if self.counters.numel() < need:
                self.counters = torch.zeros(need, dtype=torch.int32, device=dev)
        else:
            # padded by the largest leading dimension: TMA rows of the last matrix may overhang
            pad = max([int(q.mr_lds.max()) for q in (fwd_p, adj_p) if q.mr_lds is not None and len(q.mr_lds)] + [0])
            if share_arena_with is not None:
                if share_arena_with._arena_pad < pad or share_arena_with.packed.arena.shape != packed.arena.shape:
                    raise ValueError("arena layouts differ")
                self._arena_pad = share_arena_with._arena_pad
                self.arena = share_arena_with.arena
            else:
                self._arena_pad = pad
                self.arena = torch.zeros(len(packed.arena) + pad + 16, dtype=torch.complex128, device=dev)
                self.arena[: len(packed.arena)].copy_(torch.from_numpy(packed.arena))
            self.work = self.zeros(packed.work_len, torch.complex128)
            n_ctr = max(packed.fwd.n_counters, packed.adj.n_counters, 1)
            self.counters = self.zeros(n_ctr, torch.int32)
            self.ticket = self.zeros(1, torch.int64)
            self.exit_count = self.zeros(1, torch.int32)
            nmax = max(packed.n_rows, packed.n_cols, 1)
            self.x_scratch = self.zeros(nmax, torch.complex128)
            self.w_scratch = self.zeros(nmax, torch.complex128)
        self.fwd = _DeviceProgram(torch, fwd_p, dev)
        self.adj = _DeviceProgram(torch, adj_p, dev)
        d = _lib.UhmvDesc()
        d.abi_version = _lib.ABI_VERSION
        d.device = dev.index
        d.n_rows = packed.n_rows
        d.n_cols = packed.n_cols
        d.arena = self.arena.data_ptr()
        d.arena_len = len(packed.arena)
        d.work = self.work.data_ptr()
        d.work_len = packed.work_len
        d.counters = self.counters.data_ptr()
        d.ticket = self.ticket.data_ptr()
        d.exit_count = self.exit_count.data_ptr()
        d.x_scratch = self.x_scratch.data_ptr()
        d.w_scratch = self.w_scratch.data_ptr()
        d.fwd = self.fwd.struct()
        d.adj = self.adj.struct()
        self._desc = d
        handle = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(L.uhmv_plan_create(ctypes.byref(d), ctypes.byref(handle)), "uhmv_plan_create")
        self._plan = handle
        self._lock = threading.Lock()

    # ---- guarded buffers (diagnostics) ----
    _SENTINEL = {8: 0x7FF8DEADBEEF0001, 4: 0x7EADBEEF}

    def zeros(self, n, dtype):
        """A zeroed device buffer of n elements; with ``guard`` it sits between two sentinel
        bands (bit patterns: a NaN payload for 16-B / 8-B elements, 0x7EADBEEF for 4-B ones)."""
        torch = self.torch
        G = self._guard
        if G <= 0:
            return torch.zeros(max(int(n), 1), dtype=dtype, device=self.device)
        n = max(int(n), 1)
        buf = torch.empty(n + 2 * G, dtype=dtype, device=self.device)
        iv = buf.view(torch.int64) if buf.element_size() >= 8 else buf.view(torch.int32)
        iv.fill_(self._SENTINEL[iv.element_size()])
        mid = buf[G : G + n]
        mid.zero_()
        self._guards.append((buf, G, n))
        return mid

    def check_guards(self) -> list:
        """Names / offsets of sentinel elements some kernel overwrote ([] = clean)."""
        torch = self.torch
        bad = []
        torch.cuda.synchronize(self.device)
        for i, (buf, G, n) in enumerate(self._guards):
            iv = buf.view(torch.int64) if buf.element_size() >= 8 else buf.view(torch.int32)
            k = iv.numel() // buf.numel()
            want = self._SENTINEL[iv.element_size()]
            for lo, hi in ((0, G * k), ((G + n) * k, (2 * G + n) * k)):
                hit = (iv[lo:hi] != want).nonzero()
                if hit.numel():
                    bad.append((i, int(hit[0]) + lo))
        return bad

    # ---- info ----
    def launch_info(self, adjoint=False, mode=None):
        mode = mode or default_mode()
        g, s, t, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(
            _lib.lib().uhmv_plan_info(
                self._plan, int(adjoint), _MODES[mode], ctypes.byref(g), ctypes.byref(s), ctypes.byref(t), ctypes.byref(n)
            ),
            "uhmv_plan_info",
        )
        return {"grid": g.value, "smem_bytes": s.value, "threads": t.value, "stages": n.value}

    def kernel_launches(self, adjoint=False, mode=None) -> int:
        """Number of our kernel launches one matvec issues."""
        mode = mode or default_mode()
        prog = self.progs[1] if adjoint else self.progs[0]
        if prog.n_ops == 0:
            return 0
        return len(prog.phases) if mode == "phased" else 1

    def profile(self, adjoint=False, mode="bulk"):
        """Diagnostics: run one matvec with the bulk engine's per-CTA cycle counters on and
        return them summed over CTAs (see include/uhmv.h uhmv_plan_set_profile)."""
        torch = self.torch
        grid = self.launch_info(adjoint, mode)["grid"]
        buf = torch.zeros((grid, 64), dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().uhmv_plan_set_profile(self._plan, ctypes.c_void_p(buf.data_ptr())), "set_profile")
        p = self.packed
        n_in = p.n_rows if adjoint else p.n_cols
        x = torch.ones(n_in, dtype=torch.complex128, device=self.device)
        self.matvec(x, adjoint=adjoint, mode=mode)
        torch.cuda.synchronize(self.device)
        _lib.check(_lib.lib().uhmv_plan_set_profile(self._plan, None), "set_profile")
        from .packer import KIND_NAMES

        tot = buf.sum(dim=0).tolist()
        out = {"grid": grid, "p_wait_stage": tot[56], "p_wait_slot": tot[57],
               "warp_wait_data": tot[58:62], "kinds": {}}
        cats = ["wait_data", "wait_dep", "compute", "overhead", "pieces", "ops"]
        for k, name in enumerate(KIND_NAMES):
            row = tot[k * 8 : k * 8 + 6]
            if row[5]:
                out["kinds"][name] = dict(zip(cats, row))
        return out

    def trace(self, adjoint=False, x=None):
        """Diagnostics: one profiled bulk matvec with the op timeline on.  Returns a
        (n_ops, 4) int64 array {start, dependencies met, end, CTA} per op (ns, %globaltimer,
        relative to the first start) and the program's kinds."""
        torch = self.torch
        prog = self.progs[1] if adjoint else self.progs[0]
        grid = self.launch_info(adjoint, "bulk")["grid"]
        buf = torch.zeros((grid, 64), dtype=torch.int64, device=self.device)
        tr = torch.zeros((max(prog.n_ops, 1), 4), dtype=torch.int64, device=self.device)
        L = _lib.lib()
        _lib.check(L.uhmv_plan_set_profile(self._plan, ctypes.c_void_p(buf.data_ptr())), "set_profile")
        _lib.check(L.uhmv_plan_set_trace(self._plan, ctypes.c_void_p(tr.data_ptr())), "set_trace")
        p = self.packed
        n_in = p.n_rows if adjoint else p.n_cols
        if x is None:
            x = torch.ones(n_in, dtype=torch.complex128, device=self.device)
        try:
            self.matvec(x, adjoint=adjoint, mode="bulk")
            torch.cuda.synchronize(self.device)
        finally:
            L.uhmv_plan_set_trace(self._plan, None)
            L.uhmv_plan_set_profile(self._plan, None)
        t = tr.cpu().numpy()
        t0 = t[:, 0][t[:, 0] > 0].min()
        t[:, :3] -= t0
        return t, prog.kinds.copy()

    def profile_mr(self, R=64, adjoint=False):
        """Diagnostics: one multi-RHS block product with the staged engine's per-CTA cycle
        counters on (csrc/uhmv_mrtc.cuh), summed over CTAs."""
        torch = self.torch
        mr, _ = self._mr_plan()
        buf = torch.zeros((4096, 64), dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().uhmv_plan_set_profile(mr._plan, ctypes.c_void_p(buf.data_ptr())), "set_profile")
        p = self.packed
        n_in = p.n_rows if adjoint else p.n_cols
        try:
            self.matmat(torch.ones((n_in, R), dtype=torch.complex128, device=self.device), adjoint=adjoint)
            torch.cuda.synchronize(self.device)
        finally:
            _lib.check(_lib.lib().uhmv_plan_set_profile(mr._plan, None), "set_profile")
        from .packer import KIND_NAMES

        tot = buf.sum(dim=0).tolist()
        out = {"producer": dict(wait_stage=tot[0], wait_dep=tot[1], issue=tot[2], ticket_slot=tot[3]),
               "consumer_wait_op": tot[40], "kinds": {}}
        for k, name in enumerate(KIND_NAMES[:6]):
            row = tot[8 + 4 * k : 12 + 4 * k]
            if any(row):
                out["kinds"][name] = dict(zip(["wait_data", "mma", "table_flush", "s_reduce"], row))
        return out

    # ---- execution ----
    def _stream(self, stream):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def _check_out(self, out, shape):
        """The C side writes exactly prod(shape) complex128 at out.data_ptr(): refuse anything
        else (a wrong size, dtype, stride or device would be an out-of-bounds HBM write)."""
        torch = self.torch
        if (not isinstance(out, torch.Tensor) or out.dtype != torch.complex128 or out.device != self.device
                or tuple(out.shape) != tuple(shape) or not out.is_contiguous()):
            raise ValueError(f"out must be a contiguous complex128 {self.device} tensor of shape {tuple(shape)}")

    def matvec(self, x, adjoint=False, out=None, mode=None, stream=None):
        """Device API: x is a CUDA complex128 tensor (n_in,), returns/fills out (n_out,)."""
        torch = self.torch
        p = self.packed
        n_in, n_out = (p.n_rows, p.n_cols) if adjoint else (p.n_cols, p.n_rows)
        if x.shape != (n_in,) or x.dtype != torch.complex128 or x.device != self.device:
            raise ValueError(f"x must be a complex128 {self.device} tensor of shape ({n_in},)")
        x = x.contiguous()
        if out is None:
            out = torch.empty(n_out, dtype=torch.complex128, device=self.device)
        else:
            self._check_out(out, (n_out,))
        mode = mode or default_mode()
        rc = _lib.lib().uhmv_execute(
            self._plan, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), int(adjoint),
            _MODES[mode], self._stream(stream),
        )
        _lib.check(rc, "uhmv_execute")
        return out

    def matmat(self, X, adjoint=False, out=None, stream=None):
        """Multi-RHS device API on FP64 tensor cores: X (n_in, R) complex128 CUDA tensor ->
        (n_out, R).  R is padded to a multiple of 16 internally."""
        torch = self.torch
        p = self.packed
        n_in, n_out = (p.n_rows, p.n_cols) if adjoint else (p.n_cols, p.n_rows)
        if X.dim() != 2 or X.shape[0] != n_in or X.dtype != torch.complex128 or X.device != self.device:
            raise ValueError(f"X must be a complex128 {self.device} tensor of shape ({n_in}, R)")
        if out is not None:
            self._check_out(out, (n_out, X.shape[1]))
        R = X.shape[1]
        Rp = max(16, (R + 15) // 16 * 16)
        if Rp != R:
            Xp = torch.zeros((n_in, Rp), dtype=torch.complex128, device=self.device)
            Xp[:, :R] = X
        else:
            Xp = X.contiguous()
        W = torch.empty((n_out, Rp), dtype=torch.complex128, device=self.device)
        mr, work_len = self._mr_plan()
        need = work_len * Rp
        if getattr(self, "_work_mr", None) is None or self._work_mr.numel() < need:
            self._work_mr = self.zeros(need, torch.complex128)
        rc = _lib.lib().uhmv_execute_mrhs(
            mr._plan, ctypes.c_void_p(Xp.data_ptr()), ctypes.c_void_p(W.data_ptr()),
            ctypes.c_void_p(self._work_mr.data_ptr()), int(Rp), int(adjoint), self._stream(stream),
        )
        _lib.check(rc, "uhmv_execute_mrhs")
        res = W[:, :R] if Rp != R else W
        if out is not None:
            out.copy_(res)
            return out
        return res

    def matmat_host(self, X_host: np.ndarray, adjoint=False, out: np.ndarray | None = None, chunk: int | None = None,
                    stream=None):
        """Multi-RHS with host buffers (C ABI ``uhmv_matmat_host``): X_host (n_in, R) row-major
        complex128 -> (n_out, R).  The columns go in chunks of ``chunk`` whose H2D copy, DMMA
        product and D2H copy overlap on three streams (pin X_host / out for the overlap).
        R must be a multiple of ``chunk`` (a multiple of 16).  Default: 32-column chunks when R
        allows two or more (config 3: the DMMA engine at R = 16 is far below its R = 64 rate,
        measured 1.57 ms vs 2.98 ms per block; 32 columns: 1.98 ms, and the pipeline hides the
        copies -- 5.6 ms per 64-column host block vs 6.1 ms unpipelined)."""
        torch = self.torch
        p = self.packed
        n_in, n_out = (p.n_rows, p.n_cols) if adjoint else (p.n_cols, p.n_rows)
        if X_host.dtype != np.complex128 or not X_host.flags.c_contiguous or X_host.ndim != 2 or X_host.shape[0] != n_in:
            raise ValueError(f"X_host must be a C-contiguous complex128 array of shape ({n_in}, R)")
        R = X_host.shape[1]
        if chunk is None:
            chunk = 32 if (R % 32 == 0 and R > 32) else R
        if chunk % 16 or R % chunk:
            raise ValueError("R must be a multiple of chunk, chunk a multiple of 16")
        if out is None:
            out = np.empty((n_out, R), dtype=np.complex128)
        elif out.dtype != np.complex128 or not out.flags.c_contiguous or out.shape != (n_out, R):
            raise ValueError(f"out must be a C-contiguous complex128 array of shape ({n_out}, {R})")
        mr, work_len = self._mr_plan()
        key = (n_in, n_out, chunk, work_len)
        if getattr(self, "_mmh", None) is None or self._mmh[0] != key:
            dev = self.device
            self._mmh = (key, torch.empty(2 * max(n_in, n_out) * chunk, dtype=torch.complex128, device=dev),
                         torch.empty(2 * max(n_in, n_out) * chunk, dtype=torch.complex128, device=dev),
                         torch.zeros(work_len * chunk, dtype=torch.complex128, device=dev))
        _key, xd, wd, work = self._mmh
        with self._lock, torch.cuda.device(self.device):
            rc = _lib.lib().uhmv_matmat_host(
                mr._plan, ctypes.c_void_p(X_host.ctypes.data), ctypes.c_void_p(out.ctypes.data), int(R),
                ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(wd.data_ptr()), ctypes.c_void_p(work.data_ptr()),
                int(chunk), int(adjoint), self._stream(stream),
            )
        _lib.check(rc, "uhmv_matmat_host")
        return out

    def _mr_plan(self):
        """The multi-RHS plan: the same arena with whole-leaf NEAR / FAR ops
        (packer.MR_ROWS; ``UHMV_MR_ROWS=0`` keeps the single-RHS programs)."""
        if getattr(self, "_mr", None) is None:
            from .packer import MR_ROWS

            p = self.packed
            rows = int(os.environ.get("UHMV_MR_ROWS", MR_ROWS))
            can = p.geo is not None or (rows, rows) in p.rechunked
            if rows > 0 and can and p.world == 1 and self.progs == (p.fwd, p.adj):
                fwd, adj, work_len = p.programs(rows_per_chunk=rows, far_rows=rows)
                self._mr = (DeviceOperator(p, device=self.device, programs=(fwd, adj), share_with=self), work_len)
            else:
                self._mr = (self, p.work_len)
        return self._mr

    def execute_phases(self, x, out, adjoint, lo, hi, stream=None):
        rc = _lib.lib().uhmv_execute_phases(
            self._plan, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), int(adjoint),
            int(lo), int(hi), self._stream(stream),
        )
        _lib.check(rc, "uhmv_execute_phases")

    def attach_io(self) -> bool:
        """Build, upload and attach the host-I/O programs (packer ``io_programs``) once: with
        them ``matvec_host`` on pinned buffers can run ONE launch that reads x and writes w over
        PCIe itself.  False when the operator has none (or this is a partitioned / re-chunked
        plan)."""
        if getattr(self, "_io", None) is not None:
            return bool(self._io)
        self._io = ()
        p = self.packed
        if p.world != 1 or self.progs != (p.fwd, p.adj) or os.environ.get("UHMV_HOST_IO", "1") == "0":
            return False
        fwd, adj = p.io_programs()
        if fwd is None and adj is None:
            return False
        torch = self.torch
        dev = [_DeviceProgram(torch, q, self.device) if q is not None else None for q in (fwd, adj)]
        n_ctr = max([q.n_counters for q in (fwd, adj) if q is not None] + [1])
        ctr = torch.zeros(n_ctr, dtype=torch.int32, device=self.device)
        structs = [d.struct() if d is not None else _lib.UhmvProgram() for d in dev]  # empty = copy path
        with self.torch.cuda.device(self.device):
            _lib.check(_lib.lib().uhmv_plan_set_io(self._plan, ctypes.byref(structs[0]), ctypes.byref(structs[1]),
                                                   ctypes.c_void_p(ctr.data_ptr())), "uhmv_plan_set_io")
        self._io = (dev, ctr, structs, (fwd is not None, adj is not None))
        self._io_path = {}  # per direction: the path the C plan is set to
        self._io_tune = {False: ([], []), True: ([], [])}  # per direction: (io times, copy times)
        self._io_use = {}
        return True

    def _set_path(self, adjoint: bool, io: bool):
        if self._io_path.get(adjoint) != io:
            _lib.check(_lib.lib().uhmv_plan_set_host_path(self._plan, int(adjoint), int(io)), "set_host_path")
            self._io_path[adjoint] = io

    def matvec_host(self, x_host: np.ndarray, adjoint=False, out: np.ndarray | None = None, mode=None, stream=None,
                    host_io=None):
        """End-to-end C-ABI call with host buffers, then a stream synchronize.
        Pinned buffers (e.g. ``tensor.pin_memory().numpy()``) can take the host-I/O launch (x read
        and w written over PCIe inside the kernel, overlapping it); pageable ones always take
        H2D copy, kernel, D2H copy.  ``host_io``: None = with pinned buffers, time both paths on
        the first calls of each direction (graph replays of each) and keep the faster (the
        host-I/O launch pays PCIe latency at the start of the kernel, which loses on small
        operators); True / False = force."""
        p = self.packed
        n_in, n_out = (p.n_rows, p.n_cols) if adjoint else (p.n_cols, p.n_rows)
        if x_host.dtype != np.complex128 or not x_host.flags.c_contiguous:
            x_host = np.ascontiguousarray(x_host, dtype=np.complex128)
        if x_host.shape != (n_in,):
            raise ValueError(f"x must have shape ({n_in},)")
        if out is None:
            out = np.empty(n_out, dtype=np.complex128)
        elif out.dtype != np.complex128 or not out.flags.c_contiguous or out.shape != (n_out,):
            raise ValueError(f"out must be a contiguous complex128 array of shape ({n_out},)")
        mode = mode or default_mode()
        adjoint = bool(adjoint)
        with self._lock:  # the plan's path choice and the C graph cache are per-plan state
            return self._matvec_host_locked(x_host, adjoint, out, mode, stream, host_io)

    def _matvec_host_locked(self, x_host, adjoint, out, mode, stream, host_io):
        torch = self.torch
        L = _lib.lib()
        use, tuning = False, False
        if mode == "bulk" and host_io is not False and self.attach_io() and self._io[3][int(adjoint)]:
            pinned = bool(L.uhmv_host_pinned(ctypes.c_void_p(x_host.ctypes.data))) and bool(
                L.uhmv_host_pinned(ctypes.c_void_p(out.ctypes.data)))
            if host_io:
                use = True
            elif adjoint in self._io_use:
                use = self._io_use[adjoint]
            elif pinned:  # only pinned calls can take the host-I/O launch: only they are timed
                t_io, t_cp = self._io_tune[adjoint]
                use, tuning = len(t_io) <= len(t_cp), True
            self._set_path(adjoint, use)
        elif getattr(self, "_io", None):
            self._set_path(adjoint, False)
        t0 = time.perf_counter()
        # (the device switch costs ~10 us of host time per call: only when needed)
        if torch.cuda.current_device() == self.device.index:
            rc = L.uhmv_matvec_host(
                self._plan, ctypes.c_void_p(x_host.ctypes.data), ctypes.c_void_p(out.ctypes.data),
                int(adjoint), _MODES[mode], self._stream(stream),
            )
        else:
            with torch.cuda.device(self.device):
                rc = L.uhmv_matvec_host(
                    self._plan, ctypes.c_void_p(x_host.ctypes.data), ctypes.c_void_p(out.ctypes.data),
                    int(adjoint), _MODES[mode], self._stream(stream),
                )
        dt = time.perf_counter() - t0
        _lib.check(rc, "uhmv_matvec_host")
        if tuning and L.uhmv_plan_last_host_path(self._plan, int(adjoint)) == int(use):
            t_io, t_cp = self._io_tune[adjoint]
            (t_io if use else t_cp).append(dt)
            if len(t_io) >= 4 and len(t_cp) >= 4:  # the first call of each path captures its graph
                self._io_use[adjoint] = min(t_io[1:]) < min(t_cp[1:])
        return out

    def matvec_array(self, v: np.ndarray, adjoint=False, dtype=np.complex128) -> np.ndarray:
        """The drop-in's host call (``matvec_uh(u, ndarray)``): ``v`` of any dtype and layout is
        copied (and promoted) into a plan-owned pinned staging vector, the pinned host call runs
        (captured graph, §5b of DESIGN.md), and the result is copied into a NEW array of
        ``dtype`` (real part for a real result type, as uniform.py:495 implies)."""
        p = self.packed
        n_in, n_out = (p.n_rows, p.n_cols) if adjoint else (p.n_cols, p.n_rows)
        if v.shape != (n_in,):
            raise ValueError(f"x must have shape ({n_in},)")
        adjoint = bool(adjoint)
        with self._lock:
            st = getattr(self, "_staging", None)
            if st is None:
                torch = self.torch
                st = {}
                for adj in (False, True):
                    a, b = (p.n_rows, p.n_cols) if adj else (p.n_cols, p.n_rows)
                    st[adj] = (torch.empty(max(a, 1), dtype=torch.complex128).pin_memory(),
                               torch.empty(max(b, 1), dtype=torch.complex128).pin_memory())
                self._staging = st
            xs, ws = st[adjoint]
            xs_np, ws_np = xs.numpy()[:n_in], ws.numpy()[:n_out]
            torch = self.torch
            # host copies in and out: torch's multi-threaded copy for the common dtypes on vectors
            # of >= 1 MB (config 3: drop-in 1574 -> 1624 matvec/s); below that its thread-pool
            # start-up costs more than it saves (config 1: 11439 -> 9866), so NumPy copies
            big = n_in >= _TORCH_COPY_MIN and n_out >= _TORCH_COPY_MIN
            tin = _TORCH_DTYPES.get(np.dtype(v.dtype)) if big else None
            if tin is not None and v.flags.c_contiguous and v.flags.writeable:
                xs[:n_in].copy_(torch.from_numpy(v))
            else:
                np.copyto(xs_np, v, casting="unsafe" if np.iscomplexobj(v) else "same_kind")
            self._matvec_host_locked(xs_np, adjoint, ws_np, default_mode(), None, None)
            tout = _TORCH_DTYPES.get(np.dtype(dtype)) if big else None
            if tout is not None:
                res = torch.empty(n_out, dtype=tout)
                res.copy_(ws[:n_out] if np.issubdtype(dtype, np.complexfloating) else ws[:n_out].real)
                return res.numpy()  # a NEW array (it owns the tensor's storage)
            if np.issubdtype(dtype, np.complexfloating):
                return ws_np.astype(dtype, copy=True)
            return ws_np.real.astype(dtype, copy=True)

    def host_io_choice(self, adjoint=False):
        """Which path matvec_host settled on for pinned buffers: True host-I/O, False copy,
        None not decided (or unavailable)."""
        return getattr(self, "_io_use", {}).get(bool(adjoint))

    def close(self):
        mr = getattr(self, "_mr", None)
        if mr is not None and mr[0] is not self:
            mr[0].close()
        self._mr = None
        if getattr(self, "_plan", None):
            _lib.lib().uhmv_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
