"""P0 packer: UniformHMatrix -> one aligned complex128 arena + two op programs.

Replaces the dict-walking of ``matvec_uh`` (reference uniform.py:505-548) with flat,
device-resident tables.  Reads the operator duck-typed through the attributes the
reference defines (uniform.py:90-117, clustering.py:31-209); every slab is copied,
because fresh bases from the reference are non-contiguous views.

Arena (complex128, every slab 128-byte aligned = 8 elements):
  V_t   column bases, row-major |t| x l_t            (reference layout, uniform.py:43-53)
  U_s   row bases,    row-major |s| x l_s
  X_s   per row cluster s, row-major l_s x K_s: the coupling of every admissible block
        b in row(s), factorized blocks first (s_x,b: l_s x k_b) then product blocks
        (S_b = s_x s_y^H: l_s x l_t).  Per block the cheaper form is stored
        (min(k_b (l_s+l_t), l_s l_t)).
  Y_t   per column cluster t, row-major l_t x K'_t: s_y,b of the factorized blocks in col(t)
  D_b   dense leaves, row-major, grouped by row leaf

Programs (one forward, one adjoint) are lists of *ops*; every op is
  gather input runs -> smem vector xin
  sum of GEMV segments over arena/work slabs  (N: out[r] += M[r,:] xin,
                                               H: out[j] += sum_r conj(M[r,j]) xin[r],
                                               S: out[j] += sum_r M[r,j])
  scatter the smem output vector to output runs (store or add)
and carries a wait list / signal list of dependency counters for the fused
persistent launch.  The forward program (reference phase 1/2, uniform.py:509-548):
  P1   per in-leaf chunk:  partial[t] = V_t[chunk]^H x[chunk]  for all ancestors t
  NEAR per out-leaf chunk: w[chunk]  = sum_b D_b[chunk,:] x[c_b]          (store)
  RED  per t:              y_t = sum of partials                      (fixed order)
  U    per t:              u_t = Y_t^H y_t   (the stage_b vectors, uniform.py:518)
  Z    per s:              z_s = X_s [u_b | y_t]_b  (row-cluster owned, no atomics)
  FAR  per out-leaf chunk: w[chunk] += sum_{s ancestor} U_s[chunk,:] z_s
The adjoint program mirrors it with the roles of row/column swapped and conjugate
transposes taken on the fly (uniform.py:498-503, :543-544) -- no slab is stored twice.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["PackedOperator", "Program", "pack", "MODE_N", "MODE_H", "MODE_S"]

MODE_N, MODE_H, MODE_S = 0, 1, 2
BUF_ARENA, BUF_WORK, BUF_X, BUF_W = 0, 1, 2, 3
RUN_ADD = 1

OP_FIELDS = 16  # int32 per op
# op layout: n_in, n_out, in_b, in_e, seg_b, seg_e, out_b, out_e, wait_b, wait_e,
#            sig_b, sig_e, kind, pad, pad, pad
SEG_FIELDS = 8  # int64: m_off, buf, rows, cols, ld, mode, in_off, out_off
RUN_FIELDS = 5  # int64: buf, off, len, dst, flags

KIND_P1, KIND_NEAR, KIND_RED, KIND_U, KIND_Z, KIND_FAR, KIND_ZERO = range(7)
KIND_NAMES = ["P1", "NEAR", "RED", "U", "Z", "FAR", "ZERO"]

ALIGN = 8  # complex128 elements per 128 B
HCOLS_MAX = 32  # widest H/S segment (= csrc kHColsMax: 4 accumulators x 8 lanes)
ROWS_PER_CHUNK = 16  # output rows per NEAR/FAR op (= row-groups per CTA)
P1_CHUNK = 256  # max input rows per P1 op


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


@dataclass
class Program:
    """Host copy of one op program (int arrays ready for upload)."""

    ops: np.ndarray  # (n_ops, OP_FIELDS) int32
    segs: np.ndarray  # (n_segs, SEG_FIELDS) int64
    runs: np.ndarray  # (n_runs, RUN_FIELDS) int64
    waits: np.ndarray  # (n_waits, 2) int32: counter id, arrivals per matvec
    sigs: np.ndarray  # (n_sigs,) int32 counter ids
    phases: list  # [(op_begin, op_end)] for the phased (multi-launch) mode
    fused_order: np.ndarray  # (n_ops,) int32: op index claimed by ticket i in the fused launch
    in_max: int
    out_max: int
    n_counters: int
    kinds: np.ndarray  # (n_ops,) op kind

    @property
    def n_ops(self) -> int:
        return int(self.ops.shape[0])


@dataclass
class PackedOperator:
    n_rows: int
    n_cols: int
    dtype: np.dtype
    arena: np.ndarray  # complex128
    work_len: int
    fwd: Program
    adj: Program
    n_adm: int
    n_dense: int
    bytes_alg: int  # SURVEY.md §8d operator bytes (cheapest stored form), without vectors
    bytes_arena: int
    storage: dict = field(default_factory=dict)


def _leaves_under(tree):
    """For every node id: (first leaf position, one-past-last) into the DFS leaf list."""
    nodes = tree.nodes
    leaves = []
    span = [None] * len(nodes)

    def walk(i):
        n = nodes[i]
        first = len(leaves)
        if not n.children:
            leaves.append(i)
        else:
            for c in n.children:
                walk(c)
        span[i] = (first, len(leaves))

    import sys

    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 10000))
    try:
        walk(getattr(tree, "root", 0))
    finally:
        sys.setrecursionlimit(old)
    return leaves, span


def _ancestors_in(tree, leaves, span, cset):
    """For every leaf position: the clusters of ``cset`` that contain it (root to leaf)."""
    anc = [[] for _ in leaves]
    # order clusters by level so each list is root -> leaf
    for cid in sorted(cset, key=lambda c: tree.nodes[c].level):
        a, b = span[cid]
        for p in range(a, b):
            anc[p].append(cid)
    return anc


def _chunks(lo, hi, step):
    """Split [lo, hi) into near-equal chunks of at most ``step``."""
    n = hi - lo
    if n <= 0:
        return []
    k = -(-n // step)
    base, extra = divmod(n, k)
    out = []
    a = lo
    for i in range(k):
        b = a + base + (1 if i < extra else 0)
        out.append((a, b))
        a = b
    return out


def _hpanels(cols):
    return _chunks(0, cols, HCOLS_MAX)


def pack(u, *, rows_per_chunk: int = ROWS_PER_CHUNK, near_interleave=(0.4, 0.3, 0.3)) -> PackedOperator:
    """Pack a UniformHMatrix (reference object or mirror) into arena + programs."""
    bct = u.bct
    rtree, ctree = bct.row_tree, bct.col_tree
    n_rows, n_cols = bct.shape
    rnodes, cnodes = rtree.nodes, ctree.nodes

    # ---- which blocks / clusters take part (exactly what the reference walks) ----
    adm = []  # (bid, s, t) in row_map order per s
    for s in bct.row_map:
        for t in bct.row_map[s]:
            adm.append((bct.block_of[(s, t)], s, t))
    rank_r = {s: int(u.row_basis.matrices[s].shape[1]) for s in bct.row_map}
    rank_c = {t: int(u.col_basis.matrices[t].shape[1]) for t in bct.col_map}
    kb = {}
    factorized = {}
    bytes_coupling = 0
    for bid, s, t in adm:
        pair = u.coeffs[bid]
        k = int(pair.s_x.shape[1])
        kb[bid] = k
        ls, lt = rank_r[s], rank_c[t]
        fac = k * (ls + lt) < ls * lt
        factorized[bid] = fac
        bytes_coupling += min(k * (ls + lt), ls * lt)

    dense_ids = list(u.dense.keys())
    # ---- arena layout ----
    offs = {}
    cursor = 0

    def alloc(key, n):
        nonlocal cursor
        offs[key] = cursor
        cursor += _align(max(n, 0))

    for t in sorted(bct.col_map):
        alloc(("V", t), cnodes[t].size * rank_c[t])
    for s in sorted(bct.row_map):
        alloc(("U", s), rnodes[s].size * rank_r[s])
    # X_s columns: factorized blocks first, then product blocks (row_map order within)
    xcols = {}
    for s in sorted(bct.row_map):
        pos = 0
        cols = []
        for t in bct.row_map[s]:
            bid = bct.block_of[(s, t)]
            if factorized[bid]:
                cols.append((bid, t, pos, kb[bid], True))
                pos += kb[bid]
        kfac = pos
        for t in bct.row_map[s]:
            bid = bct.block_of[(s, t)]
            if not factorized[bid]:
                cols.append((bid, t, pos, rank_c[t], False))
                pos += rank_c[t]
        xcols[s] = (cols, kfac, pos)
        alloc(("X", s), rank_r[s] * pos)
    ycols = {}
    for t in sorted(bct.col_map):
        pos = 0
        cols = []
        for s in bct.col_map[t]:
            bid = bct.block_of[(s, t)]
            if factorized[bid]:
                cols.append((bid, s, pos, kb[bid]))
                pos += kb[bid]
        ycols[t] = (cols, pos)
        alloc(("Y", t), rank_c[t] * pos)
    # dense grouped by row leaf (for the forward NEAR ops), column order within
    dense_by_rleaf = {}
    dense_by_cleaf = {}
    for bid in dense_ids:
        b = bct.nodes[bid]
        dense_by_rleaf.setdefault(b.row, []).append(bid)
        dense_by_cleaf.setdefault(b.col, []).append(bid)
    for r in dense_by_rleaf:
        dense_by_rleaf[r].sort(key=lambda bid: cnodes[bct.nodes[bid].col].lo)
    for c in dense_by_cleaf:
        dense_by_cleaf[c].sort(key=lambda bid: rnodes[bct.nodes[bid].row].lo)
    for r in sorted(dense_by_rleaf, key=lambda r: rnodes[r].lo):
        for bid in dense_by_rleaf[r]:
            rr, cc = bct.block_shape(bid)
            alloc(("D", bid), rr * cc)

    arena = np.zeros(max(cursor, ALIGN), dtype=np.complex128)

    def put(key, mat):
        m = np.asarray(mat)
        if m.size:
            arena[offs[key] : offs[key] + m.size] = m.reshape(-1)

    for t in bct.col_map:
        put(("V", t), u.col_basis.matrices[t])
    for s in bct.row_map:
        put(("U", s), u.row_basis.matrices[s])
    for s, (cols, kfac, ktot) in xcols.items():
        ls = rank_r[s]
        if ls == 0 or ktot == 0:
            continue
        xs = np.empty((ls, ktot), dtype=np.complex128)
        for bid, t, pos, w, fac in cols:
            pair = u.coeffs[bid]
            xs[:, pos : pos + w] = pair.s_x if fac else pair.s_x @ np.conj(pair.s_y).T
        put(("X", s), xs)
    for t, (cols, ktot) in ycols.items():
        lt = rank_c[t]
        if lt == 0 or ktot == 0:
            continue
        ys = np.empty((lt, ktot), dtype=np.complex128)
        for bid, s, pos, w in cols:
            ys[:, pos : pos + w] = u.coeffs[bid].s_y
        put(("Y", t), ys)
    bytes_dense = 0
    for bid in dense_ids:
        d = u.dense[bid]
        bytes_dense += d.size
        put(("D", bid), d)

    bytes_bases = sum(cnodes[t].size * rank_c[t] for t in bct.col_map) + sum(
        rnodes[s].size * rank_r[s] for s in bct.row_map
    )
    geo = dict(
        bct=bct, rnodes=rnodes, cnodes=cnodes, rank_r=rank_r, rank_c=rank_c, kb=kb,
        factorized=factorized, xcols=xcols, ycols=ycols, offs=offs,
        dense_by_rleaf=dense_by_rleaf, dense_by_cleaf=dense_by_cleaf,
    )
    fwd, work_f = _build_program(geo, adjoint=False, rows_per_chunk=rows_per_chunk, near_interleave=near_interleave)
    adj, work_a = _build_program(geo, adjoint=True, rows_per_chunk=rows_per_chunk, near_interleave=near_interleave)
    elems_alg = bytes_bases + bytes_coupling + bytes_dense
    return PackedOperator(
        n_rows=n_rows,
        n_cols=n_cols,
        dtype=np.dtype(u._dtype),
        arena=arena,
        work_len=max(work_f, work_a, 1),
        fwd=fwd,
        adj=adj,
        n_adm=len(adm),
        n_dense=len(dense_ids),
        bytes_alg=16 * elems_alg,
        bytes_arena=16 * int(arena.size),
        storage=dict(
            bases=16 * bytes_bases,
            coupling=16 * bytes_coupling,
            dense=16 * bytes_dense,
            n_factorized=int(sum(factorized.values())),
            n_product=int(len(adm) - sum(factorized.values())),
        ),
    )


def _build_program(geo, *, adjoint: bool, rows_per_chunk: int, near_interleave):
    bct = geo["bct"]
    offs = geo["offs"]
    xcols, ycols = geo["xcols"], geo["ycols"]
    factorized = geo["factorized"]
    if adjoint:
        in_tree, out_tree = bct.row_tree, bct.col_tree
        in_map, out_map = bct.row_map, bct.col_map
        in_rank, out_rank = geo["rank_r"], geo["rank_c"]
        in_basis_key, out_basis_key = "U", "V"
        dense_by_outleaf = geo["dense_by_cleaf"]
    else:
        in_tree, out_tree = bct.col_tree, bct.row_tree
        in_map, out_map = bct.col_map, bct.row_map
        in_rank, out_rank = geo["rank_c"], geo["rank_r"]
        in_basis_key, out_basis_key = "V", "U"
        dense_by_outleaf = geo["dense_by_rleaf"]
    in_nodes, out_nodes = in_tree.nodes, out_tree.nodes

    # ---- work-buffer layout ----
    work = 0

    def walloc(n):
        nonlocal work
        o = work
        work += max(int(n), 0)
        return o

    in_leaves, in_span = _leaves_under(in_tree)
    out_leaves, out_span = _leaves_under(out_tree)
    in_anc = _ancestors_in(in_tree, in_leaves, in_span, [t for t in in_map if in_rank[t] > 0])
    out_anc = _ancestors_in(out_tree, out_leaves, out_span, [s for s in out_map if out_rank[s] > 0])

    # P1 chunks: every in-leaf split in <= P1_CHUNK rows
    p1_items = []  # (leafpos, lo, hi)
    for p, leaf in enumerate(in_leaves):
        if not in_anc[p]:
            continue
        n = in_nodes[leaf]
        for a, b in _chunks(n.lo, n.hi, P1_CHUNK):
            p1_items.append((p, a, b))
    # partial slots per in-cluster t: one per P1 chunk under t
    chunks_of = {t: [] for t in in_map}
    for idx, (p, a, b) in enumerate(p1_items):
        for t in in_anc[p]:
            chunks_of[t].append(idx)
    y_off, part_off = {}, {}
    for t in sorted(in_map, key=lambda t: in_nodes[t].lo):
        y_off[t] = walloc(in_rank[t])
    for t in sorted(in_map, key=lambda t: in_nodes[t].lo):
        nchunk = len(chunks_of[t])
        if in_rank[t] == 0:
            continue
        part_off[t] = y_off[t] if nchunk == 1 else walloc(nchunk * in_rank[t])
    # staging vectors u: forward per column cluster t (Y_t columns), adjoint per row cluster s
    # (factorized columns [0, kfac) of X_s)
    u_off, u_len = {}, {}
    for t in sorted(in_map, key=lambda t: in_nodes[t].lo):
        n = ycols[t][1] if not adjoint else xcols[t][1]
        u_len[t] = n
        u_off[t] = walloc(n)
    z_off = {}
    for s in sorted(out_map, key=lambda s: out_nodes[s].lo):
        z_off[s] = walloc(out_rank[s])

    # position of block b's staging vector inside u of its in-cluster
    u_pos = {}
    for t in in_map:
        if not adjoint:
            for bid, s, pos, w in ycols[t][0]:
                u_pos[bid] = pos
        else:
            for bid, tt, pos, w, fac in xcols[t][0]:
                if fac:
                    u_pos[bid] = pos

    # ---- counters ----
    n_ctr = 0

    def ctr():
        nonlocal n_ctr
        n_ctr += 1
        return n_ctr - 1

    c_part = {t: ctr() for t in in_map}
    c_y = {t: ctr() for t in in_map}
    c_u = {t: ctr() for t in in_map}
    c_z = {s: ctr() for s in out_map}

    phase_ops = {k: [] for k in range(7)}

    # P1: partial_t = B_in,t[chunk rows]^H x[chunk]
    for idx, (p, a, b) in enumerate(p1_items):
        segs, outs, sigs = [], [], []
        oo = 0
        for t in in_anc[p]:
            lt = in_rank[t]
            tl = in_nodes[t].lo
            for c0, c1 in _hpanels(lt):
                segs.append((offs[(in_basis_key, t)] + (a - tl) * lt + c0, BUF_ARENA, b - a, c1 - c0, lt, MODE_H, 0, oo + c0))
            slot = chunks_of[t].index(idx)
            outs.append((BUF_WORK, part_off[t] + slot * lt, lt, oo, 0))
            sigs.append(c_part[t])
            oo += lt
        phase_ops[KIND_P1].append(
            (KIND_P1, b - a, oo, [(BUF_X, a, b - a, 0, 0)], segs, outs, [], sigs, (b - a) * oo)
        )
    # RED: y_t = sum over chunk partials (skipped when the single partial is y_t itself)
    for t in in_map:
        lt = in_rank[t]
        nchunk = len(chunks_of[t])
        if lt == 0:
            continue
        waits = [(c_part[t], nchunk)]
        if nchunk <= 1:
            continue
        segs = [(part_off[t] + c0, BUF_WORK, nchunk, c1 - c0, lt, MODE_S, 0, c0) for c0, c1 in _hpanels(lt)]
        phase_ops[KIND_RED].append(
            (KIND_RED, 0, lt, [], segs, [(BUF_WORK, y_off[t], lt, 0, 0)], waits, [c_y[t]], nchunk * lt)
        )
    y_wait = {}
    for t in in_map:
        if in_rank[t] == 0:
            y_wait[t] = []
        elif len(chunks_of[t]) <= 1:
            y_wait[t] = [(c_part[t], len(chunks_of[t]))]
        else:
            y_wait[t] = [(c_y[t], 1)]
    # U: staging vectors of the factorized blocks, u_t = C_t^H y_t.  When l_t = 0 the
    # staging vectors are exact zeros (reference: (k x 0) @ (0,)), which the zero-initialised,
    # never-written work region already holds -- no op, no wait.
    u_wait = {}
    for t in in_map:
        n = u_len[t]
        lt = in_rank[t]
        u_wait[t] = []
        if n == 0 or lt == 0:
            continue
        u_wait[t] = [(c_u[t], 1)]
        if not adjoint:
            base, ld = offs[("Y", t)], ycols[t][1]
        else:
            base, ld = offs[("X", t)], xcols[t][2]
        segs = [(base + c0, BUF_ARENA, lt, c1 - c0, ld, MODE_H, 0, c0) for c0, c1 in _hpanels(n)]
        phase_ops[KIND_U].append(
            (KIND_U, lt, n, [(BUF_WORK, y_off[t], lt, 0, 0)], segs, [(BUF_WORK, u_off[t], n, 0, 0)],
             list(y_wait[t]), [c_u[t]], lt * n)
        )
    # Z: row-cluster (forward) / column-cluster (adjoint) owned coupling
    for s in out_map:
        ls = out_rank[s]
        if ls == 0:
            continue
        in_runs, segs, waits = [], [], []
        if not adjoint:
            cols, kfac, ktot = xcols[s]
            # gathered input in X_s column order: u_b for factorized, y_t for product blocks
            for bid, t, pos, w, fac in cols:
                if w == 0:
                    continue
                if fac:
                    in_runs.append((BUF_WORK, u_off[t] + u_pos[bid], w, pos, 0))
                    waits.extend(u_wait[t])
                else:
                    in_runs.append((BUF_WORK, y_off[t], w, pos, 0))
                    waits.extend(y_wait[t])
            if ktot:
                segs.append((offs[("X", s)], BUF_ARENA, ls, ktot, ktot, MODE_N, 0, 0))
            n_in = ktot
            nbytes = ls * ktot
        else:
            # adjoint: z_t = Y_t [u'_b] (N) + sum_{product b} S_b^H y'_s (H)
            cols, ktot = ycols[s]
            for bid, r, pos, w in cols:
                if w == 0:
                    continue
                in_runs.append((BUF_WORK, u_off[r] + u_pos[bid], w, pos, 0))
                waits.extend(u_wait[r])
            if ktot:
                segs.append((offs[("Y", s)], BUF_ARENA, ls, ktot, ktot, MODE_N, 0, 0))
            n_in = ktot
            nbytes = ls * ktot
            for r in out_map[s]:
                bid = bct.block_of[(r, s)]
                if factorized[bid]:
                    continue
                lr = in_rank[r]
                if lr == 0:
                    continue
                xc, kfac, kx = xcols[r]
                pos = next(p for (b2, tt, p, w, fac) in xc if b2 == bid)
                in_runs.append((BUF_WORK, y_off[r], lr, n_in, 0))
                waits.extend(y_wait[r])
                for c0, c1 in _hpanels(ls):
                    segs.append((offs[("X", r)] + pos + c0, BUF_ARENA, lr, c1 - c0, kx, MODE_H, n_in, c0))
                n_in += lr
                nbytes += lr * ls
        waits = sorted(set(waits))
        phase_ops[KIND_Z].append(
            (KIND_Z, n_in, ls, in_runs, segs, [(BUF_WORK, z_off[s], ls, 0, 0)], waits, [c_z[s]], nbytes)
        )

    # NEAR + FAR per output leaf chunk
    near_ctr = {}
    far_list = []
    for p, leaf in enumerate(out_leaves):
        n = out_nodes[leaf]
        dlist = dense_by_outleaf.get(leaf, [])
        for a, b in _chunks(n.lo, n.hi, rows_per_chunk):
            rows = b - a
            has_near = False
            if dlist:
                in_runs, segs = [], []
                pos = 0
                nbytes = 0
                for bid in dlist:
                    blk = bct.nodes[bid]
                    if not adjoint:
                        c = bct.col_tree.nodes[blk.col]
                        width = c.size
                        in_runs.append((BUF_X, c.lo, width, pos, 0))
                        segs.append((offs[("D", bid)] + (a - n.lo) * width, BUF_ARENA, rows, width, width, MODE_N, pos, 0))
                        pos += width
                        nbytes += rows * width
                    else:
                        r = bct.row_tree.nodes[blk.row]
                        width = n.size  # dense block is |r| x |c|, c = this out-leaf
                        in_runs.append((BUF_X, r.lo, r.size, pos, 0))
                        for c0, c1 in _hpanels(rows):
                            segs.append((offs[("D", bid)] + (a - n.lo) + c0, BUF_ARENA, r.size, c1 - c0, width, MODE_H, pos, c0))
                        pos += r.size
                        nbytes += rows * r.size
                cid = ctr()
                near_ctr[(a, b)] = cid
                phase_ops[KIND_NEAR].append(
                    (KIND_NEAR, pos, rows, in_runs, segs, [(BUF_W, a, rows, 0, 0)], [], [cid], nbytes)
                )
                has_near = True
            anc = out_anc[p]
            if anc:
                in_runs, segs, waits = [], [], []
                pos = 0
                for s in anc:
                    ls = out_rank[s]
                    sl = out_nodes[s].lo
                    in_runs.append((BUF_WORK, z_off[s], ls, pos, 0))
                    segs.append((offs[(out_basis_key, s)] + (a - sl) * ls, BUF_ARENA, rows, ls, ls, MODE_N, pos, 0))
                    waits.append((c_z[s], 1))
                    pos += ls
                if has_near:
                    waits.append((near_ctr[(a, b)], 1))
                far_list.append(
                    (KIND_FAR, pos, rows, in_runs, segs, [(BUF_W, a, rows, 0, RUN_ADD if has_near else 0)],
                     waits, [], rows * pos)
                )
            elif not has_near:
                phase_ops[KIND_ZERO].append((KIND_ZERO, 0, rows, [], [], [(BUF_W, a, rows, 0, 0)], [], [], 0))
    phase_ops[KIND_FAR] = far_list

    # ---- order: largest first inside each phase (reference uniform.py:505-506) ----
    for k in phase_ops:
        phase_ops[k].sort(key=lambda o: -o[-1])

    near = phase_ops[KIND_NEAR]
    f = np.cumsum([0.0] + list(near_interleave))
    f = f / f[-1]
    cut = [int(round(x * len(near))) for x in f]
    near_parts = [near[cut[i] : cut[i + 1]] for i in range(len(near_interleave))]
    while len(near_parts) < 3:
        near_parts.append([])
    # phased launches (multi-launch mode): [P1 + NEAR + ZERO] [RED] [U] [Z] [FAR]
    phased = [phase_ops[KIND_P1] + near + phase_ops[KIND_ZERO]]
    phased += [phase_ops[k] for k in (KIND_RED, KIND_U, KIND_Z, KIND_FAR)]
    # fused persistent order: every op waits only on ops that come earlier
    fused = (
        phase_ops[KIND_P1]
        + near_parts[0]
        + phase_ops[KIND_RED]
        + phase_ops[KIND_U]
        + near_parts[1]
        + phase_ops[KIND_Z]
        + near_parts[2]
        + phase_ops[KIND_ZERO]
        + phase_ops[KIND_FAR]
    )
    return _finish(phased, fused, n_ctr), work


def _finish(phased, fused, n_ctr):
    """Flatten op tuples into arrays in the phased order; the fused order is a
    permutation (``fused_order[ticket] = op index``)."""
    order = [o for ph in phased for o in ph]
    bounds = []
    a = 0
    for ph in phased:
        if ph:
            bounds.append((a, a + len(ph)))
        a += len(ph)
    index = {id(o): i for i, o in enumerate(order)}
    fused_order = np.array([index[id(o)] for o in fused], dtype=np.int32)
    assert len(fused_order) == len(order) and len(set(fused_order.tolist())) == len(order)

    n = len(order)
    ops = np.zeros((n, OP_FIELDS), dtype=np.int32)
    segs, runs, waits, sigs = [], [], [], []
    in_max = out_max = 0
    for i, (kind, n_in, n_out, in_runs, sg, out_runs, wt, sgn, _) in enumerate(order):
        in_b = len(runs)
        runs.extend(in_runs)
        in_e = len(runs)
        out_b = len(runs)
        runs.extend(out_runs)
        out_e = len(runs)
        seg_b = len(segs)
        segs.extend(_order_segments(sg))
        seg_e = len(segs)
        w_b = len(waits)
        waits.extend(wt)
        w_e = len(waits)
        s_b = len(sigs)
        sigs.extend(sgn)
        s_e = len(sigs)
        ops[i, :13] = (n_in, n_out, in_b, in_e, seg_b, seg_e, out_b, out_e, w_b, w_e, s_b, s_e, kind)
        in_max = max(in_max, n_in)
        out_max = max(out_max, n_out)
    return Program(
        ops=ops,
        segs=np.asarray(segs, dtype=np.int64).reshape(-1, SEG_FIELDS),
        runs=np.asarray(runs, dtype=np.int64).reshape(-1, RUN_FIELDS),
        waits=np.asarray(waits, dtype=np.int32).reshape(-1, 2),
        sigs=np.asarray(sigs, dtype=np.int32).reshape(-1),
        phases=bounds,
        fused_order=fused_order,
        in_max=in_max,
        out_max=out_max,
        n_counters=n_ctr,
        kinds=ops[:, 12].copy(),
    )


def _order_segments(segs):
    """N segments first (grouped by out_off/rows), then H/S groups (by out_off/cols).

    The device kernel accumulates consecutive segments that share (mode, out_off,
    rows|cols) in registers and reduces once per group; N before H/S lets N rows be
    owner-updated without a barrier (see csrc/uhmv_kernels.cu)."""
    n = [s for s in segs if s[5] == MODE_N]
    h = [s for s in segs if s[5] != MODE_N]
    n.sort(key=lambda s: (s[7], s[2]))
    h.sort(key=lambda s: (s[5], s[7], s[3]))
    return n + h
