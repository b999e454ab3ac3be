"""NumPy interpreter of a packed op program.

TEST INFRASTRUCTURE ONLY (see oracle/matvec_oracle.py header): it walks the packed
arena and op tables exactly as the CUDA kernel does, so the packer's layout can be
pinned against ``oracle_matvec_uh`` on the CPU (and the multi-rank exchange logic
exercised under gloo) without a GPU.  It is never a fallback for the product path.
"""

from __future__ import annotations

import numpy as np

from paper_2405_15573_b200.packer import (
    BUF_ARENA,
    BUF_W,
    BUF_WORK,
    BUF_X,
    MODE_H,
    MODE_N,
    MODE_NW,
    MODE_S,
    MODE_T,
    MR_FIRST,
    MR_ZERO,
    OP_PEER,
    PI_DIRECT,
    PI_XGLOBAL,
    PI_XSTAGE,
    RUN_ADD,
    RUN_ATOMIC,
    RUN_PEER,
)

__all__ = ["run_program", "vm_matvec", "vm_peer_matvec"]


def _segments(prog, i, engine):
    """(m_off, buf, rows, cols, ld, mode, in_off, out_off, x_global) of op i, as the register
    kernel (``segs``) or the bulk-copy kernel (``pieces``) sees them."""
    if engine == "segs":
        for s in prog.segs[prog.ops[i, 4] : prog.ops[i, 5]]:
            yield (*s, False)
    else:
        for m_off, ld, rows, cols, mode, in_off, out_off, info in prog.pieces[prog.ops[i, 13] : prog.ops[i, 14]]:
            buf = BUF_WORK if info & PI_DIRECT else BUF_ARENA
            yield (m_off, buf, rows, cols, ld, mode, in_off, out_off, bool(info & (PI_XGLOBAL | PI_XSTAGE)))


def run_op(prog, i, bufs, engine="segs", peers=()):
    """One op; ``peers``: the other ranks' work buffers (peer-exchange programs store their
    RUN_PEER outputs there too)."""
    n_in, n_out, in_b, in_e = (int(v) for v in prog.ops[i, :4])
    out_b, out_e = (int(v) for v in prog.ops[i, 6:8])
    xin = np.zeros(n_in, dtype=np.complex128)
    for buf, off, ln, dst, _ in prog.runs[in_b:in_e]:
        xin[dst : dst + ln] = bufs[buf][off : off + ln]
    out = np.zeros(n_out, dtype=np.complex128)
    for m_off, buf, rows, cols, ld, mode, in_off, out_off, xg in _segments(prog, i, engine):
        src = bufs[buf]
        vin = bufs[BUF_X] if xg else xin
        idx = m_off + np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]
        m = src[idx] if rows and cols else np.zeros((rows, cols), dtype=np.complex128)
        if mode == MODE_N or mode == MODE_NW:  # NW: same product, warp-per-row on the device
            out[out_off : out_off + rows] += m @ vin[in_off : in_off + cols]
        elif mode == MODE_H:
            out[out_off : out_off + cols] += np.conj(m).T @ vin[in_off : in_off + rows]
        elif mode == MODE_T:  # symmetric variant (packer_sym): transpose without conjugation
            out[out_off : out_off + cols] += m.T @ vin[in_off : in_off + rows]
        elif mode == MODE_S:
            out[out_off : out_off + cols] += m.sum(axis=0)
        else:
            raise ValueError(mode)
    for buf, off, ln, dst, flags in prog.runs[out_b:out_e]:
        if flags & (RUN_ADD | RUN_ATOMIC):
            bufs[buf][off : off + ln] += out[dst : dst + ln]
        else:
            bufs[buf][off : off + ln] = out[dst : dst + ln]
        if flags & RUN_PEER:
            for pw in peers:
                pw[off : off + ln] = out[dst : dst + ln]


def run_program(prog, arena, work, x, w, order="phased", op_range=None, engine="segs"):
    bufs = {BUF_ARENA: arena, BUF_WORK: work, BUF_X: x, BUF_W: w}
    if order == "fused":
        seq = prog.fused_order.tolist()
        done = np.zeros(prog.n_counters, dtype=np.int64)
        for i in seq:
            wb, we, sb, se = (int(v) for v in prog.ops[i, 8:12])
            for c, cnt in prog.waits[wb:we]:
                assert done[c] >= cnt, f"op {i} waits on counter {c} ({done[c]}<{cnt}): order not topological"
            run_op(prog, i, bufs, engine)
            for c in prog.sigs[sb:se]:
                done[c] += 1
    else:
        lo, hi = (0, prog.n_ops) if op_range is None else op_range
        for i in range(lo, hi):
            run_op(prog, i, bufs, engine)


def vm_matvec(packed, v, adjoint=False, order="phased", engine="segs"):
    prog = packed.adj if adjoint else packed.fwd
    n_in, n_out = (packed.n_rows, packed.n_cols) if adjoint else (packed.n_cols, packed.n_rows)
    x = np.asarray(v, dtype=np.complex128)
    assert x.shape == (n_in,)
    w = np.zeros(n_out, dtype=np.complex128)  # the launcher zeroes w (NEAR/FAR add atomically)
    work = np.zeros(packed.work_len, dtype=np.complex128)
    run_program(prog, packed.arena, work, x, w, order=order, engine=engine)
    return w


def vm_peer_matvec(packs, v, adjoint=False, engine="pieces", epochs=1):
    """Emulate the W ranks of a peer-exchange partition (``pack(..., peer=True)``) in one
    process: each rank walks its fused ticket order in turn, running ops while their waits
    are met (counters are monotonic: epoch e waits for e x count, as on the device); RUN_PEER
    outputs are stored into every rank's work buffer and OP_PEER ops signal every rank's
    counters.  A round with no progress is a deadlock (assertion).  Returns w (every rank
    adds its own rows into one zeroed vector) after ``epochs`` consecutive matvecs."""
    W = len(packs)
    progs = [p.adj if adjoint else p.fwd for p in packs]
    assert all(pr.peer for pr in progs)
    p0 = packs[0]
    n_in, n_out = (p0.n_rows, p0.n_cols) if adjoint else (p0.n_cols, p0.n_rows)
    x = np.asarray(v, dtype=np.complex128)
    assert x.shape == (n_in,)
    works = [np.zeros(p.work_len, dtype=np.complex128) for p in packs]
    ctr = [np.zeros(max(pr.n_counters, 1), dtype=np.int64) for pr in progs]
    for epoch in range(1, epochs + 1):
        w = np.zeros(n_out, dtype=np.complex128)
        seqs = [pr.fused_order.tolist() for pr in progs]
        pos = [0] * W
        while any(pos[r] < len(seqs[r]) for r in range(W)):
            progressed = False
            for r in range(W):
                pr = progs[r]
                while pos[r] < len(seqs[r]):
                    i = seqs[r][pos[r]]
                    wb, we, sb, se = (int(q) for q in pr.ops[i, 8:12])
                    if any(ctr[r][c] < epoch * cnt for c, cnt in pr.waits[wb:we]):
                        break
                    bufs = {BUF_ARENA: packs[r].arena, BUF_WORK: works[r], BUF_X: x, BUF_W: w}
                    run_op(pr, i, bufs, engine, peers=[works[q] for q in range(W) if q != r])
                    targets = range(W) if pr.ops[i, 12] & OP_PEER else (r,)
                    for c in pr.sigs[sb:se]:
                        for q in targets:
                            ctr[q][c] += 1
                    pos[r] += 1
                    progressed = True
            assert progressed, f"peer programs deadlock at tickets {pos}"
    return w


def run_op_mr(prog, i, bufs, R):
    """Multi-RHS op exactly as the device engines flush it: vectors are (len, R) blocks; the
    resolved ``mr_segs`` form groups (same mode and outputs) that are summed and flushed once
    -- fp64 add for atomic (w) runs, store for a group flagged MR_FIRST, add otherwise; the
    op's work outputs are zeroed first only when it carries MR_ZERO."""
    out_b, out_e = (int(v) for v in prog.ops[i, 6:8])
    a, b, flags = (int(v) for v in prog.mr_ranges[i])
    out_runs = prog.runs[out_b:out_e]
    if flags & MR_ZERO:
        for buf, off, ln, dst, fl in out_runs:
            if int(buf) != BUF_W:  # (w runs: atomic adds onto the zeroed W, whatever their single-RHS flags)
                bufs[int(buf)][off : off + ln] = 0

    def flush(o0, blk, first):
        for j in range(blk.shape[0]):
            o = o0 + j
            buf, off, ln, dst, fl = next(r for r in out_runs if r[3] <= o < r[3] + r[2])
            tgt = bufs[int(buf)]
            if int(buf) == BUF_W or not first:
                tgt[off + o - dst] += blk[j]
            else:
                tgt[off + o - dst] = blk[j]

    segs = [tuple(int(v) for v in q) for q in prog.mr_segs[a:b]]
    g = 0
    while g < len(segs):
        mode, o0 = segs[g][4] & 0xFF, segs[g][7]
        nout = segs[g][2] if mode == MODE_N else segs[g][3]
        e = g + 1
        while e < len(segs) and segs[e][4] & 0x1FF == segs[g][4] & 0x1FF and segs[e][7] == o0 and (segs[e][2] if mode == MODE_N else segs[e][3]) == nout:
            e += 1
        blk = np.zeros((nout, R), dtype=np.complex128)
        for m_off, ld, rows, cols, _mode, in_buf, in_abs, _o in segs[g:e]:
            if mode == MODE_S:
                src = bufs[BUF_WORK]
                for k in range(rows):
                    blk += src[m_off + k * ld : m_off + k * ld + cols]
                continue
            idx = m_off + np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]
            m = bufs[BUF_ARENA][idx]
            vin = bufs[in_buf]
            if mode == MODE_N:
                blk += m @ vin[in_abs : in_abs + cols]
            else:
                blk += np.conj(m).T @ vin[in_abs : in_abs + rows]
        flush(o0, blk, bool(segs[g][4] & MR_FIRST))
        g = e


def vm_matmat(packed, V, adjoint=False, programs=None):
    """Multi-RHS program interpreter: V (n_in, R) -> W (n_out, R).  ``programs``: a
    (fwd, adj, work_len) re-chunked pair (PackedOperator.programs) instead of fwd / adj."""
    prog = packed.adj if adjoint else packed.fwd
    work_len = packed.work_len
    if programs is not None:
        prog = programs[1] if adjoint else programs[0]
        work_len = programs[2]
    n_in, n_out = (packed.n_rows, packed.n_cols) if adjoint else (packed.n_cols, packed.n_rows)
    X = np.asarray(V, dtype=np.complex128)
    R = X.shape[1]
    assert X.shape[0] == n_in
    W = np.zeros((n_out, R), dtype=np.complex128)
    work = np.zeros((work_len, R), dtype=np.complex128)
    bufs = {BUF_ARENA: packed.arena, BUF_WORK: work, BUF_X: X, BUF_W: W}
    for i in prog.fused_order.tolist():
        run_op_mr(prog, i, bufs, R)
    return W


def run_peer_rank(pack, rank, world, work, counters, done, x, w, adjoint=False, epochs=1, lock=None,
                  jitter=None, engine="pieces", timeout_s=60.0, scale=None):
    """One rank of a peer-exchange partition, run CONCURRENTLY with the other ranks (each in
    its own process) over shared memory -- the multi-process CPU model of the device protocol
    (csrc/uhmv_bulk.cuh, PEER):
      work[q]      every rank's work buffer, shape (2, work_len_q): epoch e uses half e & 1
      counters[q]  every rank's dependency counters (monotonic: a wait for n needs n * e)
      done[q]      every rank's done-epoch flags (done[q][r] = last epoch rank r finished)
    The rank walks its fused ticket order, polling each op's waits (and, for OP_PEER ops,
    done[rank][q] >= e - 2 for every peer q, so no store lands in a half a peer still reads);
    RUN_PEER outputs go to every rank's current half; OP_PEER ops signal every rank's
    counters (under ``lock``: the device uses atomics).  ``w`` receives this rank's rows.
    ``scale(e)``: epoch e multiplies x by it (stale data of an earlier epoch then shows in
    the result); returns the list of per-epoch outputs."""
    outs = []
    import time

    prog = pack.adj if adjoint else pack.fwd
    assert prog.peer

    def wait_until(pred):
        t0 = time.time()
        while not pred():
            if time.time() - t0 > timeout_s:
                raise TimeoutError(f"rank {rank}: peer wait timed out")
            time.sleep(0.0002)

    for epoch in range(1, epochs + 1):
        half = epoch & 1
        w[:] = 0
        xe = x * scale(epoch) if scale is not None else x
        for i in prog.fused_order.tolist():
            wb, we, sb, se = (int(q) for q in prog.ops[i, 8:12])
            peer_op = bool(prog.ops[i, 12] & OP_PEER)
            for c, cnt in prog.waits[wb:we]:
                wait_until(lambda c=int(c), cnt=int(cnt): counters[rank][c] >= epoch * cnt)
            if peer_op and epoch > 2:
                for q in range(world):
                    if q != rank:
                        wait_until(lambda q=q: done[rank][q] >= epoch - 2)
            if jitter is not None:
                time.sleep(jitter.random() * 1e-4)
            bufs = {BUF_ARENA: pack.arena, BUF_WORK: work[rank][half], BUF_X: xe, BUF_W: w}
            run_op(prog, i, bufs, engine, peers=[work[q][half] for q in range(world) if q != rank])
            targets = range(world) if peer_op else (rank,)
            if se > sb:
                if lock is not None:
                    lock.acquire()
                try:
                    for c in prog.sigs[sb:se]:
                        for q in targets:
                            counters[q][int(c)] += 1
                finally:
                    if lock is not None:
                        lock.release()
        for q in range(world):
            done[q][rank] = epoch
        outs.append(w.copy())
    return outs
