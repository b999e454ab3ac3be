"""Packer of the symmetric single-triangle variant (symmetric.py; paper Remark 4.5).

Same arena + op-program machinery as packer.py, run by the same bulk-copy engine
(csrc/uhmv_bulk.cuh).  What differs is that every stored slab is streamed ONCE and used
twice: an N piece (rows of the slab times an input window) is followed by *alias* pieces
(PI_ALIAS: no copy) that re-read column sub-blocks of the same staged rows as T (symmetric,
out[j] += sum_r M[r,j] in[r]) or H (hermitian, conjugated) products -- the mirror terms.

Arena (complex128, 128-B aligned slabs):
  XS_L  leaf stacks of the ONE basis: rows of X_t of every ancestor t of leaf L, side by side
  S_b   per lower block b = (s, t) (t before s): ell_s x ell_t, contiguous, grouped by s (a block
        is staged whole, so its mirror product's register accumulators are flushed once)
  D_b   lower and diagonal dense leaves, grouped by row leaf

Program (one; the adjoint is the forward for hermitian, conj(A conj x) for symmetric):
  P1    per leaf chunk: partial_t = V_t^H x[chunk]  (T mode sym / H mode herm over XS_L)
  RED   y_t = fixed-order sum of the partials
  Z     per (cluster s, group of its lower blocks): N  p_s = sum_b S_b y_t   -> slot of s
                                                    T  q_b = M(S_b) y_s      -> slot of t
  ZSUM  z_c = fixed-order sum of c's slots (own groups, then mirrored blocks)
  FAR   per leaf chunk: w[chunk] += XS_L[chunk] [z_s ...]                   (fp64 red.add)
  NEAR  per (row leaf r, group of its lower/diag leaves): N  D x_c -> slot of r
                                                          T  M(D) x_r -> slot of c
  WSUM  w[q] += fixed-order sum of leaf q's slots                            (fp64 red.add)
Every w entry receives exactly two red.add addends (FAR, WSUM) onto zero, every slot one
store: results are bit-reproducible.  Byte accounting (``bytes_alg``): the basis is read
twice (P1 and FAR; phase 1 must finish before phase 2), every coupling and dense slab once.
"""

from __future__ import annotations

import numpy as np

from .packer import (
    ALIGN,
    BUF_ARENA,
    BUF_W,
    BUF_WORK,
    BUF_X,
    KIND_FAR,
    KIND_NEAR,
    KIND_P1,
    KIND_RED,
    KIND_Z,
    MODE_H,
    MODE_N,
    MODE_S,
    MODE_T,
    OP_DUAL,
    OP_XIN,
    P1_CHUNK,
    RUN_ATOMIC,
    STAGE_ELEMS,
    PackedOperator,
    _align,
    _ancestors_in,
    _chunks,
    _finish,
    _leaves_under,
    _seg,
    _stacks,
)
from .symmetric import lower_blocks

__all__ = ["pack_sym", "SYM_GROUP_OUT"]

SYM_GROUP_OUT = 320  # mirrored outputs per Z / NEAR op (bounds the shared-memory output vector)
FAR_ROWS = 64


def _groups(items, width, cap):
    """Consecutive groups of ``items`` whose summed ``width`` stays <= cap (>= 1 item each)."""
    out, cur, tot = [], [], 0
    for it in items:
        w = width(it)
        if cur and tot + w > cap:
            out.append(cur)
            cur, tot = [], 0
        cur.append(it)
        tot += w
    if cur:
        out.append(cur)
    return out


def pack_sym(us, *, stage_elems: int = STAGE_ELEMS, near_interleave=None,
             group_out: int = SYM_GROUP_OUT) -> PackedOperator:
    import os

    if near_interleave is None:
        near_interleave = tuple(float(v) for v in os.environ.get("UHMV_SYM_INTERLEAVE", "0.3,0.1,0.2,0.4").split(","))
    bct = us.bct
    tree = bct.row_tree
    nodes = tree.nodes
    n = nodes[getattr(tree, "root", 0)].hi
    herm = us.kind == "hermitian"
    mmode = MODE_H if herm else MODE_T  # mirror products (and P1: V_t^H = X_t^T / X_t^H)
    X = us.basis.matrices
    rank = {c: int(X[c].shape[1]) if c in X else 0 for c in set(bct.row_map) | set(bct.col_map)}
    low_adm, low_dense = lower_blocks(bct)
    lower_of = {}  # s -> [(bid, t)] lower blocks of row cluster s, row_map order
    for s in bct.row_map:
        for t in bct.row_map[s]:
            bid = bct.block_of[(s, t)]
            if bid in us.coupling and rank[s] > 0 and rank[t] > 0:
                lower_of.setdefault(s, []).append((bid, t))

    # ---- arena ----
    offs = {}
    cursor = 0

    def alloc(key, size, ld):
        nonlocal cursor
        if ld > 1:
            cursor = (cursor + ld - 1) // ld * ld
        offs[key] = cursor
        cursor += _align(max(size, 0))

    stacks = _stacks(tree, {c: None for c in rank}, rank)
    for leaf, (W, _cols) in sorted(stacks.items()):
        alloc(("XS", leaf), nodes[leaf].size * W, W)
    cwidth = {}
    for s in sorted(lower_of):
        cwidth[s] = sum(rank[t] for _b, t in lower_of[s])
        for bid, t in lower_of[s]:
            alloc(("S", bid), rank[s] * rank[t], rank[t])
    dense_by_rleaf = {}
    for bid in low_dense:
        dense_by_rleaf.setdefault(bct.nodes[bid].row, []).append(bid)
    for r in dense_by_rleaf:
        dense_by_rleaf[r].sort(key=lambda b: nodes[bct.nodes[b].col].lo)
    for r in sorted(dense_by_rleaf, key=lambda r: nodes[r].lo):
        for bid in dense_by_rleaf[r]:
            rr, cc = bct.block_shape(bid)
            alloc(("D", bid), rr * cc, cc)
    arena = np.zeros(max(cursor, ALIGN), dtype=np.complex128)
    for leaf, (W, cols) in stacks.items():
        L = nodes[leaf]
        blk = arena[offs[("XS", leaf)] : offs[("XS", leaf)] + L.size * W].reshape(L.size, W)
        for c, c0 in cols:
            blk[:, c0 : c0 + rank[c]] = X[c][L.lo - nodes[c].lo : L.hi - nodes[c].lo]
    for s, blocks in lower_of.items():
        for bid, t in blocks:
            arena[offs[("S", bid)] : offs[("S", bid)] + rank[s] * rank[t]] = np.asarray(us.coupling[bid]).reshape(-1)
    for bid in low_dense:
        d = us.dense[bid]
        arena[offs[("D", bid)] : offs[("D", bid)] + d.size] = np.asarray(d).reshape(-1)

    # ---- work layout + counters ----
    work = 0

    def walloc(k):
        nonlocal work
        o = work
        work += max(int(k), 0)
        return o

    n_ctr = 0

    def ctr():
        nonlocal n_ctr
        n_ctr += 1
        return n_ctr - 1

    leaves, span = _leaves_under(tree)
    anc = _ancestors_in(tree, leaves, span, [c for c in rank if rank[c] > 0])
    p1_items = []
    for p, leaf in enumerate(leaves):
        if anc[p]:
            for a, b in _chunks(nodes[leaf].lo, nodes[leaf].hi, P1_CHUNK):
                p1_items.append((p, a, b))
    chunks_of = {c: [] for c in rank}
    for idx, (p, a, b) in enumerate(p1_items):
        for c in anc[p]:
            chunks_of[c].append(idx)
    y_off = {c: walloc(rank[c]) for c in sorted(rank, key=lambda c: nodes[c].lo) if rank[c] > 0}
    part_off = {c: (y_off[c] if len(chunks_of[c]) == 1 else walloc(len(chunks_of[c]) * rank[c]))
                for c in y_off if chunks_of[c]}
    z_off = {c: walloc(rank[c]) for c in y_off}
    # Z groups and the slot region of every cluster: [own groups ... | mirrored blocks ...]
    zgroups = {s: _groups(blocks, lambda bt: rank[bt[1]], group_out) for s, blocks in lower_of.items()}
    mirrors_of = {c: [] for c in y_off}
    for s in sorted(lower_of, key=lambda s: nodes[s].lo):
        for bid, t in lower_of[s]:
            mirrors_of[t].append(bid)
    zslot_rows = {c: len(zgroups.get(c, [])) + len(mirrors_of[c]) for c in y_off}
    zreg = {c: walloc(zslot_rows[c] * rank[c]) for c in y_off if zslot_rows[c]}
    mirror_row = {bid: len(zgroups.get(t, [])) + i for t, bids in mirrors_of.items() for i, bid in enumerate(bids)}
    # NEAR groups and slot regions per leaf: [own groups ... | mirrored leaves ...]
    ngroups = {r: _groups(bids, lambda b: 0 if bct.nodes[b].col == r else nodes[bct.nodes[b].col].size, group_out)
               for r, bids in dense_by_rleaf.items()}
    dmirrors_of = {}
    for r in sorted(dense_by_rleaf, key=lambda r: nodes[r].lo):
        for bid in dense_by_rleaf[r]:
            c = bct.nodes[bid].col
            if c != r:
                dmirrors_of.setdefault(c, []).append(bid)
    wleaves = sorted(set(ngroups) | set(dmirrors_of), key=lambda q: nodes[q].lo)
    wslot_rows = {q: len(ngroups.get(q, [])) + len(dmirrors_of.get(q, [])) for q in wleaves}
    wreg = {q: walloc(wslot_rows[q] * nodes[q].size) for q in wleaves}
    dmirror_row = {bid: len(ngroups.get(q, [])) + i for q, bids in dmirrors_of.items() for i, bid in enumerate(bids)}

    c_part = {c: ctr() for c in y_off}
    c_y = {c: ctr() for c in y_off}
    c_zs = {c: ctr() for c in y_off}
    c_z = {c: ctr() for c in y_off}
    c_ws = {q: ctr() for q in wleaves}
    ops = {k: [] for k in range(7)}
    zsum_ops, wsum_ops = [], []

    # P1 (one op per leaf chunk, every ancestor at once)
    for idx, (p, a, b) in enumerate(p1_items):
        leaf = leaves[p]
        W, cols = stacks[leaf]
        c0 = dict(cols)
        first = c0[anc[p][0]]
        width = sum(rank[c] for c in anc[p])
        outs, sigs, oo = [], [], 0
        for c in anc[p]:
            outs.append((BUF_WORK, part_off[c] + chunks_of[c].index(idx) * rank[c], rank[c], oo, 0))
            sigs.append(c_part[c])
            oo += rank[c]
        base = offs[("XS", leaf)] + (a - nodes[leaf].lo) * W
        segs = [_seg(base + first, BUF_ARENA, b - a, width, W, mmode, 0, 0, a)]
        ops[KIND_P1].append((KIND_P1, b - a, oo, [(BUF_X, a, b - a, 0, 0)], segs, outs, [], sigs, (b - a) * oo))
    # RED
    y_wait = {}
    for c in y_off:
        k = len(chunks_of[c])
        if k <= 1:
            y_wait[c] = [(c_part[c], 1)] if k else []
            continue
        segs = [_seg(part_off[c], BUF_WORK, k, rank[c], rank[c], MODE_S, 0, 0)]
        ops[KIND_RED].append((KIND_RED, 0, rank[c], [], segs, [(BUF_WORK, y_off[c], rank[c], 0, 0)],
                              [(c_part[c], k)], [c_y[c]], k * rank[c]))
        y_wait[c] = [(c_y[c], 1)]
    # Z: one op per (s, block group): per block an N segment (S_b y_t -> own slot) whose pieces
    # are followed by alias T / H pieces (M(S_b) y_s -> the block's mirror slot)
    for s, groups in zgroups.items():
        ls = rank[s]
        for g, grp in enumerate(groups):
            k_in = sum(rank[t] for _b, t in grp)
            in_runs, waits, pos = [], list(y_wait[s]), 0
            for _b, t in grp:
                in_runs.append((BUF_WORK, y_off[t], rank[t], pos, 0))
                waits.extend(y_wait[t])
                pos += rank[t]
            in_runs.append((BUF_WORK, y_off[s], ls, pos, 0))  # y_s: the mirror products' input
            segs, outs, sigs, oo, pos = [], [(BUF_WORK, zreg[s] + g * ls, ls, 0, 0)], [c_zs[s]], ls, 0
            for bid, t in grp:
                lt = rank[t]
                segs.append(_seg(offs[("S", bid)], BUF_ARENA, ls, lt, lt, MODE_N, pos, 0) + (((0, lt, mmode, k_in, oo),),))
                outs.append((BUF_WORK, zreg[t] + mirror_row[bid] * lt, lt, oo, 0))
                sigs.append(c_zs[t])
                oo += lt
                pos += lt
            ops[KIND_Z].append((KIND_Z | OP_DUAL, k_in + ls, oo, in_runs, segs, outs, sorted(set(waits)), sigs,
                                ls * k_in))
    # ZSUM: z_c = sum of its slot rows (fixed order)
    for c in y_off:
        if not zslot_rows[c]:
            continue
        segs = [_seg(zreg[c], BUF_WORK, zslot_rows[c], rank[c], rank[c], MODE_S, 0, 0)]
        zsum_ops.append((KIND_RED, 0, rank[c], [], segs, [(BUF_WORK, z_off[c], rank[c], 0, 0)],
                         [(c_zs[c], 0)], [c_z[c]], zslot_rows[c] * rank[c]))
    # FAR: w[chunk] += XS_L[chunk] [z_s ...]
    for p, leaf in enumerate(leaves):
        cl = [c for c in anc[p] if c in zreg]
        if not cl:
            continue
        W, cols = stacks[leaf]
        c0 = dict(cols)
        L = nodes[leaf]
        for a, b in _chunks(L.lo, L.hi, FAR_ROWS):
            in_runs, waits, segs, pos = [], [], [], 0
            for c in cl:
                in_runs.append((BUF_WORK, z_off[c], rank[c], pos, 0))
                waits.append((c_z[c], 1))
                segs.append(_seg(offs[("XS", leaf)] + (a - L.lo) * W + c0[c], BUF_ARENA, b - a, rank[c], W,
                                 MODE_N, pos, 0))
                pos += rank[c]
            ops[KIND_FAR].append((KIND_FAR, pos, b - a, in_runs, segs, [(BUF_W, a, b - a, 0, RUN_ATOMIC)], waits, [],
                                  (b - a) * pos))
    # NEAR: per (row leaf r, leaf group): N D x_c -> own slot, T/H M(D) x_r -> mirror slots
    for r, groups in ngroups.items():
        R = nodes[r]
        for g, grp in enumerate(groups):
            segs, outs, sigs, oo = [], [(BUF_WORK, wreg[r] + g * R.size, R.size, 0, 0)], [c_ws[r]], R.size
            nbytes = 0
            for bid in grp:
                c = bct.nodes[bid].col
                C = nodes[c]
                alias = ()
                if c != r:
                    alias = ((0, C.size, mmode, 0, oo),)
                    outs.append((BUF_WORK, wreg[c] + dmirror_row[bid] * C.size, C.size, oo, 0))
                    sigs.append(c_ws[c])
                    oo += C.size
                segs.append(_seg(offs[("D", bid)], BUF_ARENA, R.size, C.size, C.size, MODE_N, 0, 0, C.lo) + (alias,))
                nbytes += R.size * C.size
            ops[KIND_NEAR].append((KIND_NEAR | OP_XIN | OP_DUAL, R.size, oo, [(BUF_X, R.lo, R.size, 0, 0)], segs, outs, [],
                                   sigs, nbytes))
    # WSUM: w[q] += sum of its slot rows (fixed order)
    for q in wleaves:
        Q = nodes[q]
        segs = [_seg(wreg[q], BUF_WORK, wslot_rows[q], Q.size, Q.size, MODE_S, 0, 0)]
        wsum_ops.append((KIND_RED, 0, Q.size, [], segs, [(BUF_W, Q.lo, Q.size, 0, RUN_ATOMIC)], [(c_ws[q], 0)], [],
                         wslot_rows[q] * Q.size))

    # waits count every producer of the counter
    allops = [o for k in ops for o in ops[k]] + zsum_ops + wsum_ops
    producers = {}
    for o in allops:
        for c in o[7]:
            producers[c] = producers.get(c, 0) + 1

    def fix(lst):
        return [o[:6] + ([(c, producers.get(c, 0)) for c, _n in o[6]],) + o[7:] for o in lst]

    for k in ops:
        ops[k] = sorted(fix(ops[k]), key=lambda o: -o[-1])
    zsum_ops, wsum_ops = fix(zsum_ops), fix(wsum_ops)
    near = ops[KIND_NEAR]
    f = np.cumsum([0.0] + list(near_interleave))
    f = f / f[-1]
    cut = [int(round(v * len(near))) for v in f]
    parts = [near[cut[i] : cut[i + 1]] for i in range(len(near_interleave))] + [[], [], [], []]
    # chain first (ZSUM right behind the Z ops, FAR before the last nearfield share): the
    # nearfield (no dependencies) fills the gaps, and WSUM -- which waits for every NEAR op
    # of its leaf -- closes the program
    fused = (ops[KIND_P1] + parts[0] + ops[KIND_RED] + parts[1] + ops[KIND_Z] + zsum_ops + parts[2]
             + ops[KIND_FAR] + parts[3] + wsum_ops)
    phased = [ops[KIND_P1] + near, ops[KIND_RED], ops[KIND_Z], zsum_ops + wsum_ops, ops[KIND_FAR]]
    prog = _finish(phased, fused, n_ctr, stage_elems=stage_elems, bulk_only=True)
    basis_el = sum(nodes[c].size * rank[c] for c in rank)
    coup_el = sum(rank[s] * cwidth[s] for s in cwidth)  # (the per-block slabs, without alignment)
    dense_el = sum(np.asarray(us.dense[b]).size for b in low_dense)
    return PackedOperator(
        n_rows=n, n_cols=n, dtype=np.dtype(us._dtype), arena=arena, work_len=max(work, 1), fwd=prog, adj=prog,
        n_adm=2 * len(low_adm), n_dense=2 * len(low_dense) - sum(1 for b in low_dense if bct.nodes[b].row == bct.nodes[b].col),
        bytes_alg=16 * (2 * basis_el + coup_el + dense_el), bytes_arena=16 * int(arena.size),
        storage=dict(basis=16 * basis_el, coupling=16 * coup_el, dense=16 * dense_el, kind=us.kind, symmetric=True),
    )
