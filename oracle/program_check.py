"""Static bounds validator of packed op programs (a compute-sanitizer stand-in).

TEST INFRASTRUCTURE ONLY (see oracle/matvec_oracle.py header).  compute-sanitizer is closed
on this GPU pool (profiles/r02/sanitizer_closed.txt), so out-of-bounds accesses are ruled out
here instead: every address the CUDA engines derive from a program -- bulk copies out of the
arena (csrc/uhmv_bulk.cuh producer), x windows carried in a stage, shared-memory stage
offsets, xin / outv indices of the consumers, gather / scatter runs, dependency counters,
multi-RHS segments (csrc/uhmv_mrtc.cuh) -- is recomputed the way the kernels decode it and
checked against the buffer it lands in.  The device-side counterpart is the UHMV_CHECKS
build (tests/test_gpu_checked.py), which asserts the same bounds inside the kernels.
"""

from __future__ import annotations

import numpy as np

from paper_2405_15573_b200.packer import (
    BUF_ARENA,
    BUF_W,
    BUF_WORK,
    BUF_X,
    BULK_HCOLS_MAX,
    MODE_H,
    MODE_N,
    MODE_NW,
    MODE_S,
    MODE_T,
    PI_ALIAS,
    PI_BEGIN,
    PI_DIRECT,
    PI_END,
    PI_XSTAGE,
    RUN_ATOMIC,
    RUN_PEER,
)

__all__ = ["check_program", "check_packed"]

BUF_HOSTW = 4


class ProgramError(AssertionError):
    pass


def _fail(msg):
    raise ProgramError(msg)


def _check_cover(runs, n, what, op):
    """The consumers locate a vector position with a binary search over runs sorted by dst
    (uhmv_bulk.cuh find_run): the runs must tile [0, n) in order."""
    pos = 0
    for r in runs:
        if int(r[3]) != pos:
            _fail(f"op {op}: {what} runs do not tile [0, {n}) (gap/overlap at {pos}, next dst {int(r[3])})")
        pos += int(r[2])
    if pos != n:
        _fail(f"op {op}: {what} runs cover {pos} of {n}")


def check_program(prog, *, arena_len, arena_pad, work_len, n_in_vec, n_out_vec):
    """Raise ProgramError on the first out-of-bounds address any engine would derive."""
    ops = prog.ops
    n_ops = ops.shape[0]
    n_runs, n_pcs = prog.runs.shape[0], prog.pieces.shape[0]
    stage = int(prog.stage_elems)
    lens = {BUF_WORK: work_len, BUF_X: n_in_vec, BUF_W: n_out_vec}
    fo = np.sort(np.asarray(prog.fused_order))
    if not np.array_equal(fo, np.arange(n_ops)):
        _fail("fused_order is not a permutation of the ops")
    if len(prog.waits) and (prog.waits[:, 0].min() < 0 or prog.waits[:, 0].max() >= prog.n_counters):
        _fail("wait counter out of range")
    if len(prog.sigs) and (prog.sigs.min() < 0 or prog.sigs.max() >= prog.n_counters):
        _fail("signal counter out of range")
    for i in range(n_ops):
        n_in, n_out, in_b, in_e, seg_b, seg_e, out_b, out_e, w_b, w_e, s_b, s_e, kind, pc_b, pc_e, xin_len = (
            int(v) for v in ops[i])
        if not (0 <= in_b <= in_e == out_b <= out_e <= n_runs):
            _fail(f"op {i}: run range")
        if not (0 <= pc_b <= pc_e <= n_pcs and 0 <= w_b <= w_e <= len(prog.waits) and 0 <= s_b <= s_e <= len(prog.sigs)):
            _fail(f"op {i}: piece / wait / signal range")
        if n_out > prog.out_max or xin_len > prog.xin_max or n_in > prog.in_max:
            _fail(f"op {i}: vector larger than the launch's shared-memory sizing")
        ins = prog.runs[in_b:in_e]
        outs = prog.runs[out_b:out_e]
        _check_cover(ins, n_in, "input", i)
        _check_cover(outs, n_out, "output", i)
        for buf, off, ln, dst, fl in list(ins) + list(outs):
            buf, off, ln = int(buf), int(off), int(ln)
            if buf not in lens:
                _fail(f"op {i}: run buffer {buf}")
            if off < 0 or off + ln > lens[buf]:
                _fail(f"op {i}: run [{off}, {off + ln}) outside buffer {buf} of {lens[buf]}")
            if int(fl) & RUN_PEER and buf != BUF_WORK:
                _fail(f"op {i}: peer run outside the work buffer")
        for buf, off, ln, dst, fl in outs:
            if int(buf) == BUF_X:
                _fail(f"op {i}: writes x")
            if int(fl) & RUN_ATOMIC and int(buf) not in (BUF_W, BUF_WORK):
                _fail(f"op {i}: atomic run into buffer {int(buf)}")
        if kind & 128:  # OP_DRAIN: its drain descriptor sits right behind the output runs
            if out_e >= n_runs or int(prog.runs[out_e][0]) != BUF_HOSTW:
                _fail(f"op {i}: drain descriptor missing")
            d = prog.runs[out_e]
            if int(d[1]) < 0 or int(d[1]) + int(d[2]) > n_out_vec or int(d[3]) >= prog.n_counters:
                _fail(f"op {i}: drain descriptor out of range")
        # ---- bulk-copy engine pieces ----
        open_stage = False
        fill = 0
        for j in range(pc_b, pc_e):
            m_off, ld, rows, cols, mode, in_off, out_off, info = (int(v) for v in prog.pieces[j])
            if rows <= 0 or cols <= 0 or rows >= 1 << 15 or cols >= 1 << 16:
                _fail(f"op {i} piece {j}: shape {rows}x{cols} does not fit the compressed descriptor")
            if mode not in (MODE_N, MODE_H, MODE_S, MODE_NW, MODE_T):
                _fail(f"op {i} piece {j}: mode {mode}")
            if mode in (MODE_H, MODE_S, MODE_T) and cols > BULK_HCOLS_MAX:
                _fail(f"op {i} piece {j}: {cols} H columns exceed the register slots")
            # outputs (outv) and inputs (xin or the stage's x window)
            nout = rows if mode in (MODE_N, MODE_NW) else cols
            if out_off < 0 or out_off + nout > n_out:
                _fail(f"op {i} piece {j}: outputs [{out_off}, {out_off + nout}) of {n_out}")
            span = cols if mode in (MODE_N, MODE_NW) else rows
            if info & PI_DIRECT:
                if mode != MODE_S:
                    _fail(f"op {i} piece {j}: direct piece not an S reduction")
                if m_off < 0 or m_off + (rows - 1) * ld + cols > work_len:
                    _fail(f"op {i} piece {j}: direct work rows outside the work buffer")
                continue
            if info & PI_XSTAGE:
                if in_off < 0 or in_off + span > n_in_vec:
                    _fail(f"op {i} piece {j}: x window [{in_off}, {in_off + span}) of {n_in_vec}")
            elif kind & 1024:  # OP_XWIN: the input is gathered window by window (xin_len each)
                if mode not in (MODE_N, MODE_NW) or in_off < 0 or in_off + span > n_in or span > xin_len:
                    _fail(f"op {i} piece {j}: windowed input [{in_off}, {in_off + span}) of {n_in} (window {xin_len})")
            elif mode != MODE_S and (in_off < 0 or in_off + span > xin_len):
                _fail(f"op {i} piece {j}: xin [{in_off}, {in_off + span}) of {xin_len}")
            if m_off < 0 or m_off + (rows - 1) * ld + cols > arena_len:
                _fail(f"op {i} piece {j}: arena rows [{m_off}, {m_off + (rows - 1) * ld + cols}) of {arena_len}")
            if ld < cols:
                _fail(f"op {i} piece {j}: ld {ld} < cols {cols}")
            smem = info & 0xFFFFFF
            if info & PI_ALIAS:  # re-reads staged rows of the piece before it (row stride in [32,56))
                if not open_stage or info & (PI_BEGIN | PI_XSTAGE) or mode not in (MODE_H, MODE_T):
                    _fail(f"op {i} piece {j}: alias piece outside a stage or of mode {mode}")
                stride = (info >> 32) & 0xFFFFFF
                if in_off >= 1 << 16 or stride >= 1 << 16 or smem >= 1 << 16:
                    _fail(f"op {i} piece {j}: alias fields do not fit the compressed descriptor")
                if smem + (rows - 1) * stride + cols > fill or cols > stride:
                    _fail(f"op {i} piece {j}: alias rows beyond the stage data")
                if info & PI_END:
                    open_stage = False
                continue
            xw = span if info & PI_XSTAGE else 0
            if smem + rows * cols + xw > stage:
                _fail(f"op {i} piece {j}: stage elements [{smem}, {smem + rows * cols + xw}) of {stage}")
            if info & PI_BEGIN:
                if open_stage:
                    _fail(f"op {i} piece {j}: stage begins inside an open stage")
                open_stage = True
                fill = (info >> 32) & 0xFFFFFF
                if fill > stage or fill <= 0:
                    _fail(f"op {i} piece {j}: stage fill {fill}")
            elif not open_stage:
                _fail(f"op {i} piece {j}: staged piece outside a stage")
            if smem + rows * cols + xw > fill:
                _fail(f"op {i} piece {j}: piece beyond the stage's expected bytes")
            if info & PI_END:
                open_stage = False
        if open_stage:
            _fail(f"op {i}: stage left open at the end of the op")
    # ---- multi-RHS segments (DMMA engine, TMA boxes over the arena) ----
    if prog.mr_segs is not None and len(prog.mr_segs):
        for i in range(n_ops):
            b, e, _fl = (int(v) for v in prog.mr_ranges[i])
            n_out = int(ops[i, 1])
            for m_off, ld, rows, cols, mode, in_buf, in_abs, out_off in prog.mr_segs[b:e]:
                m_off, ld, rows, cols, in_abs, out_off = (int(v) for v in (m_off, ld, rows, cols, in_abs, out_off))
                md = int(mode) & 0xFF
                if md == MODE_S:
                    if m_off < 0 or m_off + (rows - 1) * ld + cols > work_len:
                        _fail(f"op {i}: mr S segment outside the work buffer")
                    continue
                if m_off < 0 or m_off + (rows - 1) * ld + cols > arena_len + arena_pad:
                    _fail(f"op {i}: mr segment outside the padded arena")
                span = cols if md == MODE_N else rows
                if int(in_buf) not in lens or in_abs < 0 or in_abs + span > lens[int(in_buf)]:
                    _fail(f"op {i}: mr input [{in_abs}, {in_abs + span}) outside buffer {int(in_buf)}")
                nout = rows if md == MODE_N else cols
                if out_off < 0 or out_off + nout > n_out:
                    _fail(f"op {i}: mr outputs [{out_off}, {out_off + nout}) of {n_out}")


def check_packed(packed, extra_programs=()):
    """Every program of a pack (both directions, launch-B halves, host-I/O and the
    multi-RHS re-chunked programs when present) against the pack's buffer sizes."""
    pad = max([int(q.mr_lds.max()) for q in (packed.fwd, packed.adj) if q.mr_lds is not None and len(q.mr_lds)] + [0])
    arena_len = len(packed.arena)
    progs = []
    for adj, p in ((False, packed.fwd), (True, packed.adj)):
        progs.append((adj, p, packed.work_len))
        if p.part_b is not None:
            progs.append((adj, p.part_b, packed.work_len))
    for adj, p, wl in extra_programs:
        progs.append((adj, p, wl))
    for adj, p, wl in progs:
        n_in, n_out = (packed.n_rows, packed.n_cols) if adj else (packed.n_cols, packed.n_rows)
        check_program(p, arena_len=arena_len, arena_pad=pad, work_len=wl, n_in_vec=n_in, n_out_vec=n_out)
    return len(progs)
