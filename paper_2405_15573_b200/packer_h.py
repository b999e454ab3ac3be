"""Packer for the H-matrix product ``matvec_h`` (reference hmatrix.py:143-184, paper Alg 4).

Same arena + op-program format as :mod:`packer` (so the same sm_100a engines run it), but
every admissible block carries its own bases (SVDForm U_b diag(sigma_b) V_b^H,
lowrank.py:51-64).  Stored per block (128-B aligned, contiguous):
  W_b = V_b diag(sigma_b)   |t| x k_b   (sigma folded in: the product needs only sigma V^H x)
  U_b                       |s| x k_b
  D_b                       dense leaves, as for the uniform format
Forward: P1 per column-leaf chunk: partial_b = W_b[chunk]^H x[chunk] for every block whose
column cluster contains the chunk; RED: y_b = sum of partials; FAR per row-leaf chunk:
w[chunk] += sum_b U_b[chunk,:] y_b; NEAR: w[chunk] += D_b x.  The adjoint swaps the roles
(P1 over U_b, FAR over W_b: V diag(sigma) (U^H x)).  No coupling stage -- which is exactly
what the uniform format trades for smaller shared bases.
"""

from __future__ import annotations

import os

import numpy as np

from .packer import (
    BUF_ARENA,
    BUF_W,
    BUF_WORK,
    BUF_X,
    KIND_FAR,
    KIND_NEAR,
    KIND_P1,
    KIND_RED,
    MODE_H,
    MODE_N,
    MODE_NW,
    MODE_S,
    OP_XWIN,
    P1_CHUNK,
    PI_XSTAGE,
    ROWS_PER_CHUNK,
    RUN_ATOMIC,
    STAGE_ELEMS,
    PackedOperator,
    _align,
    _assign_tmaps,
    _chunks,
    _finish,
    _leaves_under,
    _seg,
)

__all__ = ["pack_h"]

P1_MAX_OUT = 512  # output entries per P1 op (bounds the consumers' shared-memory vector)
H_PANEL = 256  # H/S column panel of the bulk pieces (config 3: 1.24 ms at 512, 1.15 ms at 256)


def pack_h(h, *, rows_per_chunk: int | None = None, stage_elems: int | None = None,
           near_interleave=(0.35, 0.1, 0.2, 0.35)) -> PackedOperator:
    import os

    if rows_per_chunk is None:
        rows_per_chunk = int(os.environ.get("UHMV_ROWS_PER_CHUNK", ROWS_PER_CHUNK))
    if stage_elems is None:
        stage_elems = int(os.environ.get("UHMV_STAGE_ELEMS", STAGE_ELEMS))
    bct = h.bct
    n_rows, n_cols = bct.shape
    rnodes, cnodes = bct.row_tree.nodes, bct.col_tree.nodes
    adm = [b for b in sorted(h.admissible) if h.admissible[b].rank > 0]
    kb = {b: int(h.admissible[b].rank) for b in adm}
    offs, cursor = {}, 0

    def alloc(key, n, ld):  # start at a multiple of the leading dimension (packer.alloc)
        nonlocal cursor
        if ld > 1:
            cursor = (cursor + ld - 1) // ld * ld
        offs[key] = cursor
        cursor += _align(n)

    # leaf-stacked factors (as packer.py stacks cluster bases): for every column leaf, the
    # rows of W_b of all blocks whose column cluster contains it side by side; for every row
    # leaf, the rows of U_b likewise -- P1 and FAR of a leaf chunk read one long-row matrix
    cleaves, cspan = _leaves_under(bct.col_tree)
    rleaves, rspan = _leaves_under(bct.row_tree)
    wstack = _block_stacks(cleaves, cspan, adm, kb, lambda b: bct.nodes[b].col, lambda c: cnodes[c].level)
    ustack = _block_stacks(rleaves, rspan, adm, kb, lambda b: bct.nodes[b].row, lambda c: rnodes[c].level)
    for leaf, (w, _cols) in sorted(wstack.items()):
        alloc(("WS", leaf), cnodes[leaf].size * w, w)
    for leaf, (w, _cols) in sorted(ustack.items()):
        alloc(("US", leaf), rnodes[leaf].size * w, w)
    dense_by_rleaf, dense_by_cleaf = {}, {}
    for bid in h.dense:
        blk = bct.nodes[bid]
        dense_by_rleaf.setdefault(blk.row, []).append(bid)
        dense_by_cleaf.setdefault(blk.col, []).append(bid)
    for r in dense_by_rleaf:
        dense_by_rleaf[r].sort(key=lambda bid: cnodes[bct.nodes[bid].col].lo)
    for c in dense_by_cleaf:
        dense_by_cleaf[c].sort(key=lambda bid: rnodes[bct.nodes[bid].row].lo)
    for r in sorted(dense_by_rleaf, key=lambda r: rnodes[r].lo):
        for bid in dense_by_rleaf[r]:
            rr, cc = bct.block_shape(bid)
            alloc(("D", bid), rr * cc, cc)
    arena = np.zeros(max(cursor, 8), dtype=np.complex128)
    elems = 0
    fac = {}
    for b in adm:
        f = h.admissible[b]
        wmat = np.asarray(f.V, dtype=np.complex128) * np.asarray(f.sigma, dtype=np.float64)[None, :]
        um = np.asarray(f.U, dtype=np.complex128)
        fac[b] = (wmat, um)
        elems += wmat.size + um.size
    for key, stacks, nodes, which, cl in (("WS", wstack, cnodes, 0, lambda b: bct.nodes[b].col),
                                          ("US", ustack, rnodes, 1, lambda b: bct.nodes[b].row)):
        for leaf, (w, cols) in stacks.items():
            L = nodes[leaf]
            blk = arena[offs[(key, leaf)] : offs[(key, leaf)] + L.size * w].reshape(L.size, w)
            for b, c0 in cols:
                lo = nodes[cl(b)].lo
                blk[:, c0 : c0 + kb[b]] = fac[b][which][L.lo - lo : L.hi - lo]
    dense_elems = 0
    for bid, d in h.dense.items():
        arena[offs[("D", bid)] : offs[("D", bid)] + d.size] = np.asarray(d).reshape(-1)
        dense_elems += d.size
    geo = dict(bct=bct, adm=adm, kb=kb, offs=offs, dense_by_rleaf=dense_by_rleaf, dense_by_cleaf=dense_by_cleaf,
               wstack=wstack, ustack=ustack)
    kw = dict(rows_per_chunk=rows_per_chunk, stage_elems=stage_elems, near_interleave=near_interleave,
              far_rows=int(os.environ.get("UHMV_FAR_ROWS_H", 64)))
    # windowed FAR inputs pay off on large operators (config 3: 0.818 -> 0.893 of HBM; config 2,
    # 1 GB, is latency-bound and 4 % slower with them)
    kw["xwin"] = XWIN if 16 * (elems + dense_elems) >= 2e9 else 0
    fwd, work_f = _build_h(geo, adjoint=False, **kw)
    adj, work_a = _build_h(geo, adjoint=True, **kw)
    _assign_tmaps([fwd, adj])
    # reference storage_report (hmatrix.py:187-208) counts k (m + n + 1); sigma is folded here
    return PackedOperator(
        n_rows=n_rows, n_cols=n_cols, dtype=np.dtype(h._dtype), arena=arena,
        work_len=max(work_f, work_a, 1), fwd=fwd, adj=adj, n_adm=len(h.admissible),
        n_dense=len(h.dense), bytes_alg=16 * (elems + dense_elems), bytes_arena=16 * int(arena.size),
        storage=dict(bases=16 * elems, coupling=0, dense=16 * dense_elems, format="H"),
    )


def _block_stacks(leaves, span, adm, kb, clus, level):
    """{leaf: (width, [(block, column offset)])}: blocks whose cluster ``clus(b)`` contains the
    leaf, grouped by that cluster (root to leaf, blocks of one cluster in ``adm`` order) -- so
    the per-cluster vectors of all its blocks are contiguous in every stack."""
    per = [[] for _ in leaves]
    for b in sorted(adm, key=lambda b: (level(clus(b)), clus(b), b)):
        a, e = span[clus(b)]
        for p in range(a, e):
            per[p].append(b)
    out = {}
    for p, leaf in enumerate(leaves):
        cols, w = [], 0
        for b in per[p]:
            cols.append((b, w))
            w += kb[b]
        if w:
            out[leaf] = (w, cols)
    return out


def _build_h(geo, *, adjoint, rows_per_chunk, stage_elems, near_interleave, far_rows=64, xwin=0):
    bct, adm, kb, offs = geo["bct"], geo["adm"], geo["kb"], geo["offs"]
    if adjoint:
        in_tree, out_tree = bct.row_tree, bct.col_tree
        in_key, out_key = "US", "WS"
        in_stacks, out_stacks = geo["ustack"], geo["wstack"]
        dense_by_outleaf = geo["dense_by_cleaf"]

        def in_c(b):
            return bct.nodes[b].row

        def out_c(b):
            return bct.nodes[b].col
    else:
        in_tree, out_tree = bct.col_tree, bct.row_tree
        in_key, out_key = "WS", "US"
        in_stacks, out_stacks = geo["wstack"], geo["ustack"]
        dense_by_outleaf = geo["dense_by_rleaf"]

        def in_c(b):
            return bct.nodes[b].col

        def out_c(b):
            return bct.nodes[b].row
    in_nodes, out_nodes = in_tree.nodes, out_tree.nodes
    in_leaves, in_span = _leaves_under(in_tree)
    out_leaves, out_span = _leaves_under(out_tree)
    in_blocks = [[] for _ in in_leaves]  # blocks whose input cluster contains the leaf
    out_blocks = [[] for _ in out_leaves]
    for b in adm:
        a, e = in_span[in_c(b)]
        for p in range(a, e):
            in_blocks[p].append(b)
        a, e = out_span[out_c(b)]
        for p in range(a, e):
            out_blocks[p].append(b)

    work = 0

    def walloc(n):
        nonlocal work
        o = work
        work += int(n)
        return o

    n_ctr = 0

    def ctr():
        nonlocal n_ctr
        n_ctr += 1
        return n_ctr - 1

    # Per-cluster vectors: the blocks of an input cluster t (col(t) forward) are one group of
    # adjacent stack columns, so P1 writes each multi-chunk t's partials as ONE run
    # (part_base[t] + chunk * K_t) and RED sums them per cluster (one S op of nchunk x K_t);
    # y is laid out grouped by OUTPUT cluster s, so a FAR op gathers one run per ancestor s.
    in_groups, out_groups = {}, {}
    for b in sorted(adm):
        in_groups.setdefault(in_c(b), []).append(b)
        out_groups.setdefault(out_c(b), []).append(b)
    y_off = {}
    for sc in sorted(out_groups, key=lambda c: (out_nodes[c].level, c)):
        for b in out_groups[sc]:
            y_off[b] = walloc(kb[b])
    K = {t: sum(kb[b] for b in bl) for t, bl in in_groups.items()}
    boff = {}  # block -> offset inside its input cluster's vector
    for t, bl in in_groups.items():
        o = 0
        for b in bl:
            boff[b] = o
            o += kb[b]
    # P1 items: (leafpos, lo, hi, block group); groups are runs of adjacent stack columns
    items = []
    for p, leaf in enumerate(in_leaves):
        bl = [b for b, _c in in_stacks[leaf][1]] if leaf in in_stacks else []
        if not bl:
            continue
        n = in_nodes[leaf]
        groups, cur, tot = [], [], 0
        for b in bl:
            if cur and tot + kb[b] > P1_MAX_OUT:
                groups.append(cur)
                cur, tot = [], 0
            cur.append(b)
            tot += kb[b]
        groups.append(cur)
        for a, e in _chunks(n.lo, n.hi, P1_CHUNK):
            for grp in groups:
                items.append((p, a, e, grp))
    chunk_sets = {t: set() for t in in_groups}
    for p, a, e, grp in items:
        for t in {in_c(b) for b in grp}:
            chunk_sets[t].add((a, e))
    chunks = {t: sorted(cs) for t, cs in chunk_sets.items()}
    chunk_idx = {t: {ae: i for i, ae in enumerate(cs)} for t, cs in chunks.items()}
    part_base = {t: walloc(len(cs) * K[t]) for t, cs in sorted(chunks.items()) if len(cs) > 1}
    c_part = {t: ctr() for t in in_groups}  # P1 ops touching t (its partials / its single-chunk y)
    c_y = {t: ctr() for t in in_groups}  # RED of a multi-chunk t
    n_touch = {t: 0 for t in in_groups}
    ops = {k: [] for k in range(7)}
    for idx, (p, a, e, grp) in enumerate(items):
        segs, outs, sigs = [], [], []
        oo = 0
        leaf = in_leaves[p]
        W, cols = in_stacks[leaf]
        c0 = dict(cols)[grp[0]]
        i = 0
        while i < len(grp):  # one run per (cluster, partial row), or per block into y
            t = in_c(grp[i])
            j = i
            while j < len(grp) and in_c(grp[j]) == t:
                j += 1
            if t in part_base:
                k_run = sum(kb[b] for b in grp[i:j])
                outs.append((BUF_WORK, part_base[t] + chunk_idx[t][(a, e)] * K[t] + boff[grp[i]], k_run, oo, 0))
                oo += k_run
            else:
                for b in grp[i:j]:
                    outs.append((BUF_WORK, y_off[b], kb[b], oo, 0))
                    oo += kb[b]
            sigs.append(c_part[t])
            n_touch[t] += 1
            i = j
        base = offs[(in_key, leaf)] + (a - in_nodes[leaf].lo) * W
        segs.append(_seg(base + c0, BUF_ARENA, e - a, oo, W, MODE_H, 0, 0, a))
        ops[KIND_P1].append((KIND_P1, e - a, oo, [(BUF_X, a, e - a, 0, 0)], segs, outs, [], sigs, (e - a) * oo))
    y_wait = {}
    for t, bl in in_groups.items():
        if t not in part_base:
            y_wait[t] = (c_part[t], n_touch[t])
            continue
        nchunk = len(chunks[t])
        outs = [(BUF_WORK, y_off[b], kb[b], boff[b], 0) for b in bl]
        ops[KIND_RED].append(
            (KIND_RED, 0, K[t], [], [_seg(part_base[t], BUF_WORK, nchunk, K[t], K[t], MODE_S, 0, 0)],
             outs, [(c_part[t], n_touch[t])], [c_y[t]], nchunk * K[t])
        )
        y_wait[t] = (c_y[t], 1)
    for p, leaf in enumerate(out_leaves):
        n = out_nodes[leaf]
        dlist = dense_by_outleaf.get(leaf, [])
        near_chunks = _chunks(n.lo, n.hi, rows_per_chunk) if not adjoint else [(n.lo, n.hi)]
        for a, e in near_chunks:
            if not dlist:
                continue
            rows = e - a
            in_runs, segs, pos, nbytes = [], [], 0, 0
            for bid in dlist:
                blk = bct.nodes[bid]
                if not adjoint:
                    c = bct.col_tree.nodes[blk.col]
                    in_runs.append((BUF_X, c.lo, c.size, pos, 0))
                    segs.append(_seg(offs[("D", bid)] + (a - n.lo) * c.size, BUF_ARENA, rows, c.size, c.size, MODE_N, pos, 0, c.lo))
                    pos += c.size
                    nbytes += rows * c.size
                else:
                    r = bct.row_tree.nodes[blk.row]
                    in_runs.append((BUF_X, r.lo, r.size, pos, 0))
                    segs.append(_seg(offs[("D", bid)], BUF_ARENA, r.size, n.size, n.size, MODE_H, pos, 0, r.lo))
                    pos += r.size
                    nbytes += r.size * n.size
            ops[KIND_NEAR].append((KIND_NEAR, pos, rows, in_runs, segs, [(BUF_W, a, rows, 0, RUN_ATOMIC)], [], [], nbytes))
        bl = out_blocks[p]
        if not bl:
            continue
        for a, e in _chunks(n.lo, n.hi, far_rows):  # each FAR op gathers the whole y stack once
            rows = e - a
            in_runs, segs, waits, pos = [], [], [], 0
            W, cols = out_stacks[leaf]
            for b, _c in cols:  # stack order: grouped by output cluster, y grouped alike
                k = kb[b]
                if in_runs and in_runs[-1][1] + in_runs[-1][2] == y_off[b]:
                    r0 = in_runs[-1]
                    in_runs[-1] = (r0[0], r0[1], r0[2] + k, r0[3], r0[4])
                else:
                    in_runs.append((BUF_WORK, y_off[b], k, pos, 0))
                waits.append(y_wait[in_c(b)])
                pos += k
            assert W == pos
            segs.append(_seg(offs[(out_key, leaf)] + (a - n.lo) * W, BUF_ARENA, rows, W, W, MODE_N, 0, 0))
            ops[KIND_FAR].append(
                (KIND_FAR, pos, rows, in_runs, segs, [(BUF_W, a, rows, 0, RUN_ATOMIC)], sorted(set(waits)), [], rows * pos)
            )
    for k in ops:
        ops[k].sort(key=lambda o: -o[-1])
    near = ops[KIND_NEAR]
    f = np.cumsum([0.0] + list(near_interleave))
    f = f / f[-1]
    cut = [int(round(x * len(near))) for x in f]
    parts = [near[cut[i] : cut[i + 1]] for i in range(len(near_interleave))]
    while len(parts) < 4:
        parts.append([])
    phased = [ops[KIND_P1] + near, ops[KIND_RED], ops[KIND_FAR]]
    fused = ops[KIND_P1] + parts[0] + ops[KIND_RED] + parts[1] + parts[2] + parts[3] + ops[KIND_FAR]
    # 256-column H panels (more rows per stage) measured best for the wide per-block stacks
    prog = _finish(phased, fused, n_ctr, stage_elems=stage_elems, h_panel=H_PANEL)
    return _window_inputs(prog, xwin), work


XWIN = int(os.environ.get("UHMV_XWIN_H", 704))  # FAR input window (complex) -- 0: gather whole inputs


def _window_inputs(prog, xw):
    """FAR ops gather the y of every block of every ancestor (~1750 complex at config 3), which
    at 16 B each would cut the bulk engine to 2 CTAs/SM.  Ops whose input exceeds ``xw`` and
    whose pieces all read it as N / NW rows (in nondecreasing order) are flagged OP_XWIN: the
    kernel gathers ``xw`` elements at a time, re-gathering when a piece runs past the window
    (csrc/uhmv_bulk.cuh, uhmv_bulk_xwin_kernel).  Field 15 becomes the window length."""
    if xw <= 0:
        return prog
    ops = prog.ops
    any_w = False
    for i in range(prog.n_ops):
        n_in, xin_len = int(ops[i, 0]), int(ops[i, 15])
        if xin_len <= xw:
            continue
        pcs = prog.pieces[ops[i, 13] : ops[i, 14]]
        modes = set(int(m) for m in pcs[:, 4])
        spans = pcs[:, 3]
        if not modes <= {MODE_N, MODE_NW} or (pcs[:, 7] & PI_XSTAGE).any() or int(spans.max()) > xw:
            continue
        if (np.diff(pcs[:, 5]) < 0).any():  # windows move forward only
            continue
        ops[i, 15] = xw
        ops[i, 12] |= OP_XWIN
        any_w = True
    if any_w:
        prog.xin_max = int(ops[:, 15].max())
        prog.xwin = True
    return prog
