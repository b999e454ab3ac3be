"""P0 packer: UniformHMatrix -> one aligned complex128 arena + two op programs.

Replaces the dict walk of ``matvec_uh`` (reference uniform.py:505-548) with flat,
device-resident tables.  Reads the operator duck-typed through the attributes the
reference defines (uniform.py:90-117, clustering.py:31-209); every slab is copied,
because fresh bases from the reference are non-contiguous views.

Arena (complex128, every slab 128-byte aligned = 8 elements, every slab contiguous):
  V_t   column bases, row-major |t| x l_t            (reference layout, uniform.py:43-53)
  U_s   row bases,    row-major |s| x l_s
  F_s   per row cluster s, row-major l_s x K_s: s_x,b of the *factorized* blocks of row(s)
  S_b   per *product* block, row-major l_s x l_t, S_b = s_x s_y^H (uniform.py:67-68)
  Y_t   per column cluster t, row-major l_t x K'_t: s_y,b of the factorized blocks of col(t)
  D_b   dense leaves, row-major, grouped by row leaf
Per block the cheaper form is stored (min(k_b (l_s+l_t), l_s l_t)).

Programs (one forward, one adjoint) are lists of *ops*.  Every op
  gathers its work-buffer inputs (y / u / z vectors) into a shared-memory vector xin,
  sums GEMV *segments* streamed from the arena
      N: out[r] += M[r,:] . in        H: out[j] += sum_r conj(M[r,j]) in[r]
      S: out[j] += sum_r M[r,j]       (the fixed-order reduction of partial vectors)
  (``in`` is xin, or x itself read straight from HBM/L2 for the P1 and NEAR ops),
  scatters its output vector (store or add), and carries wait / signal lists of
  dependency counters for the fused persistent launch.
Forward program (reference phase 1 / phase 2, uniform.py:509-548):
  P1   per in-leaf chunk:  partial[t] = V_t[chunk]^H x[chunk]  for all ancestors t
  NEAR per out-leaf chunk: w[chunk]  = sum_b D_b[chunk,:] x[c_b]           (store)
  RED  per t:              y_t = sum of its partials                    (fixed order)
  U    per t:              u_t = Y_t^H y_t   -- the stage_b vectors of uniform.py:518
  Z    per s:              z_s = F_s [u_b] + sum_product S_b y_t  (row-cluster owned)
  FAR  per out-leaf chunk: w[chunk] += sum_{s ancestor} U_s[chunk,:] z_s
The adjoint program mirrors it with rows/columns swapped and conjugate transposes taken
on the fly (uniform.py:498-503, :543-544) -- no slab is stored twice.

Two device encodings of the same segments are emitted:
  ``segs``   for the register-streaming kernel (H segments split in <= 32-column panels);
  ``pieces`` for the bulk-copy (TMA engine) kernel: each segment cut into row ranges
             packed into shared-memory stages of STAGE_ELEMS complex128 (16 KiB).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["PackedOperator", "Program", "pack", "MODE_N", "MODE_H", "MODE_S"]

MODE_N, MODE_H, MODE_S = 0, 1, 2
MODE_NW = 3  # bulk-kernel piece mode: an N piece of a wide-row op (one warp per row)
MODE_T = 4  # out[j] += sum_r M[r,j] in[r]: H without the conjugation (symmetric variant, packer_sym)
WIDE_COLS = int(os.environ.get("UHMV_WIDE_COLS", 288))  # an op whose N segments all have rows this long (<= 4 rows per stage) runs them warp-per-row
BUF_ARENA, BUF_WORK, BUF_X, BUF_W = 0, 1, 2, 3
RUN_ADD = 1  # out run: read-modify-write add (single writer)
RUN_ATOMIC = 2  # out run: fp64 red.add -- w is zeroed first; <= 2 addends per entry
RUN_PEER = 4  # out run (peer-exchange programs): y/u data also stored into every peer's work
OP_PEER = 16  # op field 12 flag (peer-exchange programs): the op writes peer data and
#               signals its counters on every rank (kind = field 12 & 7)
# host-I/O programs (uhmv_matvec_host with pinned buffers: x read and w written over PCIe
# inside the kernel, no separate H2D / D2H copies)
OP_XHOST = 32  # P1 op: gathers its x window from the host buffer and stores it into device x
OP_XWAIT = 64  # NEAR op: its x windows come from device x -> the producer waits for them first
OP_DRAIN = 128  # NEAR / FAR op: the last op finishing an output leaf copies w[leaf] to the host
OP_XIN = 256  # op gathers its x runs into xin although its N pieces carry x windows (packer_sym NEAR)
OP_DUAL = 512  # packer_sym Z / NEAR: N pieces + alias T / H pieces with disjoint outputs (no barrier between)
OP_XWIN = 1024  # op gathers its input window by window (field 15 = window length, field 0 = total)
BUF_HOSTW = 4  # drain descriptor run (after the op's out runs): lo, len, counter, expected count

OP_FIELDS = 16  # int32 per op
# op layout: n_in, n_out, in_b, in_e, seg_b, seg_e, out_b, out_e, wait_b, wait_e,
#            sig_b, sig_e, kind, pc_b, pc_e, xin_len
SEG_FIELDS = 8  # int64: m_off, buf, rows, cols, ld, mode, in_off, out_off
RUN_FIELDS = 5  # int64: buf, off, len, dst, flags
PIECE_FIELDS = 8  # int64: m_off, ld, rows, cols, mode, in_off, out_off, info
MR_FIELDS = 8  # int64: m_off, ld, rows, cols, mode, in_buf, in_abs (element index), out_off
MR_FIRST = 1 << 8  # mode-field flag: first group writing its outputs (flush stores, no read-add)
MR_TMAP_SHIFT = 16  # mode-field bits 16..: index into Program.mr_lds (TMA tensor map of that ld)
MR_RANGE_FIELDS = 3  # int32 per op: mr_segs begin, end, flags
MR_ZERO = 1  # op flag: some output position is written by no group -- zero the outputs first
# piece info bits: [0,24) smem element offset in its stage, 24 stage_begin, 25 stage_end,
# 26 direct (no stage: coherent loads from the work buffer), 27 input read from x directly,
# 28 x window carried in the stage behind the matrix rows (in_off = its x index),
# [32,56) elements of the stage (on stage_begin pieces)
# 29 alias: no copy -- the piece re-reads a sub-block of the stage data of the N piece before it
# (its smem row stride in bits [32,56)); m_off / ld still address the arena (VM, checker)
PI_BEGIN, PI_END, PI_DIRECT, PI_XGLOBAL, PI_XSTAGE = 1 << 24, 1 << 25, 1 << 26, 1 << 27, 1 << 28
PI_ALIAS = 1 << 29

KIND_P1, KIND_NEAR, KIND_RED, KIND_U, KIND_Z, KIND_FAR, KIND_ZERO = range(7)
KIND_NAMES = ["P1", "NEAR", "RED", "U", "Z", "FAR", "ZERO"]

ALIGN = 8  # complex128 elements per 128 B
HCOLS_MAX = 32  # widest H/S segment of the register kernel (= csrc kHColsMax)
ROWS_PER_CHUNK = 16  # output rows per NEAR op (= consumer row-groups: one row each)
MR_ROWS = 80  # multi-RHS programs: NEAR / FAR output rows per op (= mrtc kNP, one pass)
FAR_ROWS = 64  # output rows per FAR op (4 register slots of 16 row-groups)
P1_CHUNK = 256  # max input rows per P1 op
# adjoint NEAR: output columns per op (default: the whole leaf; 40- / 27-column panels measured
# 1.36x / 1.59x slower at config 3 -- strided per-row copies make the producer the bottleneck)
ADJ_NEAR_COLS = int(os.environ.get("UHMV_ADJ_NEAR_COLS", 1 << 30))
STAGE_ELEMS = 1408  # default complex128 per shared-memory stage (22 KiB: 16 x 80 dense + x window)
BULK_NCOLS_MAX = int(os.environ.get("UHMV_NCOLS_MAX", 640))  # widest N piece row (two rows + x window still fit a stage)
NW_COLS = int(os.environ.get("UHMV_NW_COLS", 640))  # widest panel of a warp-per-row op (sweeps: 352/176 slower)
# Stored form of an admissible block: factorized (s_x, s_y: k_b (l_s + l_t) elements, one more
# phase -- the U ops -- in the forward chain) iff k_b (l_s + l_t) < FACTOR_BIAS * l_s l_t, else
# the product S_b = s_x s_y^H.  1.0 is the byte minimum.
FACTOR_BIAS = 1.0
FACTOR_BIAS_SMALL = 0.5  # operators under 1 GB (pack(): the forward chain loses its U phase for most blocks)
NOSPLIT = float(os.environ.get("UHMV_NOSPLIT", 0.3))  # see _pieces: largest stage fraction left empty instead of cutting an N segment
BULK_HCOLS_MAX = 512  # widest H/S piece of the bulk kernel (= csrc bulk::kSlots x 128 consumers)
# work splitting of the farfield chain ops across CTAs (output entries per op)
SPLIT_DEFAULTS = {"p1_out": 1 << 30, "u_cols": 1 << 30, "z_rows": 1 << 30, "far_rows": ROWS_PER_CHUNK}


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


@dataclass
class Program:
    """Host copy of one op program (int arrays ready for upload)."""

    ops: np.ndarray  # (n_ops, OP_FIELDS) int32
    segs: np.ndarray  # (n_segs, SEG_FIELDS) int64  (register kernel)
    pieces: np.ndarray  # (n_pieces, PIECE_FIELDS) int64  (bulk-copy kernel)
    runs: np.ndarray  # (n_runs, RUN_FIELDS) int64
    waits: np.ndarray  # (n_waits, 2) int32: counter id, arrivals per matvec
    sigs: np.ndarray  # (n_sigs,) int32 counter ids
    phases: list  # [(op_begin, op_end)] for the phased (multi-launch) mode
    fused_order: np.ndarray  # (n_ops,) int32: op index claimed by ticket i in the fused launch
    in_max: int  # largest gathered input (register kernel: all inputs staged)
    xin_max: int  # largest work-buffer input (bulk kernel: x is read in place)
    out_max: int
    n_counters: int
    kinds: np.ndarray  # (n_ops,) op kind
    zero_output: bool = True  # the launcher zeroes w before this program (NEAR/FAR add into it)
    arena_elems: int = 0  # complex128 arena elements the program streams (roofline bytes / 16)
    part_b: "Program | None" = None  # multi-GPU: the program launched after the y/u exchange
    stage_elems: int = STAGE_ELEMS  # bulk kernel stage size the pieces were packed for
    mr_segs: np.ndarray | None = None  # (n, MR_FIELDS) int64: multi-RHS segments, one input source each
    mr_ranges: np.ndarray | None = None  # (n_ops, 3) int32: mr_segs range + MR_ZERO flag of every op
    mr_lds: np.ndarray | None = None  # int64 leading dimensions the mr segments read (one TMA map each)
    peer: bool = False  # multi-GPU peer-exchange program: ONE launch per rank, y/u stored into
    #                     the peers' work buffers and counters signalled across ranks (RUN_PEER)
    host_io: bool = False  # host-I/O program (OP_XHOST / OP_XWAIT / OP_DRAIN ops)
    w_order: bool = False  # ordered output: NEAR stores, FAR waits for the leaf's NEAR ops and adds (no memset of w)
    bulk_only: bool = False  # T-mode / alias pieces (packer_sym): only the bulk engine runs it
    xwin: bool = False  # windowed-input ops (packer_h FAR, OP_XWIN): the bulk engine's xwin kernel

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
    rank: int = 0
    world: int = 1
    part: dict | None = None
    exchange: dict = field(default_factory=dict)  # per direction: (ex_off, ex_len) block layout
    geo: dict | None = field(default=None, repr=False)  # index structure, for re-chunked programs
    build_kw: dict | None = field(default=None, repr=False)
    rechunked: dict = field(default_factory=dict, repr=False)  # (rows, far_rows) -> (fwd, adj, work_len)
    io: tuple | None = field(default=None, repr=False)  # cached io_programs()

    def io_programs(self):
        """(fwd, adj) host-I/O programs of this single-GPU pack (``_build_program(host_io=True)``:
        x read from / w drained to pinned host buffers inside the kernel), cached; (None, None)
        when the operator's structure does not allow it (an input leaf without a P1 op, an
        output leaf without NEAR / FAR ops)."""
        if self.io is None:
            if self.geo is None or self.world != 1:
                self.io = (None, None)
            else:
                kw = dict(self.build_kw, host_io=True)
                fwd, work_f, _ = _build_program(self.geo, adjoint=False, **kw)
                adj, work_a, _ = _build_program(self.geo, adjoint=True, **kw)
                assert max(work_f, work_a, 1) <= self.work_len
                self.io = (fwd, adj)
        return self.io

    def for_rank(self, rank: int, world: int, peer: bool = False) -> "PackedOperator":
        """The same arena with the programs of one rank of a ``world``-way partition (what
        ``pack(u, rank=, world=, peer=)`` returns, without re-copying the slabs)."""
        import dataclasses

        if self.geo is None:
            raise ValueError("re-partitioning needs the pack's index structure")
        bct = self.geo["bct"]
        part = None
        if world > 1:
            part = _partition(self.geo, world, rank)
        kw = dict(self.build_kw, part=part, peer=bool(peer and world > 1))
        fwd, work_f, ex_f = _build_program(self.geo, adjoint=False, **kw)
        adj, work_a, ex_a = _build_program(self.geo, adjoint=True, **kw)
        _assign_tmaps([fwd, adj] + [q.part_b for q in (fwd, adj) if q.part_b is not None])
        return dataclasses.replace(
            self, fwd=fwd, adj=adj, work_len=max(work_f, work_a, 1), rank=rank, world=world, part=part,
            exchange={"fwd": ex_f, "adj": ex_a}, build_kw=kw, rechunked={}, io=None,
        )

    def programs(self, *, rows_per_chunk: int, far_rows: int):
        """(fwd, adj, work_len): the same operator and arena with NEAR / FAR ops re-chunked
        (the multi-RHS engine wants whole-leaf output blocks).  Single-GPU only; cached (and
        saved by packed_io) per chunking."""
        key = (int(rows_per_chunk), int(far_rows))
        if key in self.rechunked:
            return self.rechunked[key]
        if self.geo is None or self.world != 1:
            raise ValueError("re-chunking needs a single-GPU pack with its index structure")
        kw = dict(self.build_kw)
        kw["rows_per_chunk"] = rows_per_chunk
        kw["split"] = dict(kw["split"], far_rows=far_rows)
        kw["w_order"] = False  # the multi-RHS engine adds into a zeroed W
        fwd, work_f, _ = _build_program(self.geo, adjoint=False, **kw)
        adj, work_a, _ = _build_program(self.geo, adjoint=True, **kw)
        _assign_tmaps([fwd, adj])
        self.rechunked[key] = (fwd, adj, max(work_f, work_a, 1))
        return self.rechunked[key]


def _leaves_under(tree):
    """DFS leaf list and, for every node id, its (first, one-past-last) leaf position."""
    nodes = tree.nodes
    leaves = []
    span = [None] * len(nodes)
    stack = [(getattr(tree, "root", 0), False)]
    first = {}
    while stack:
        i, done = stack.pop()
        n = nodes[i]
        if done:
            span[i] = (first[i], len(leaves))
            continue
        first[i] = len(leaves)
        if not n.children:
            leaves.append(i)
            span[i] = (first[i], len(leaves))
            continue
        stack.append((i, True))
        for c in reversed(n.children):
            stack.append((c, False))
    return leaves, span


def _stacks(tree, cmap, rank):
    """Leaf-stacked basis layout: {leaf: (W, [(cluster, column offset)])} over the clusters of
    ``cmap`` with rank > 0 that contain the leaf, root to leaf."""
    leaves, span = _leaves_under(tree)
    anc = _ancestors_in(tree, leaves, span, [c for c in cmap if rank[c] > 0])
    out = {}
    for p, leaf in enumerate(leaves):
        cols, w = [], 0
        for c in anc[p]:
            cols.append((c, w))
            w += rank[c]
        if w:
            out[leaf] = (w, cols)
    return out


def unstack_basis(packed_arena, geo, which: str, c: int):
    """Reassemble cluster basis ``c`` (``which`` = "V" column, "U" row) from the leaf stacks
    (test / inspection helper)."""
    bct = geo["bct"]
    tree, stacks, key = (bct.col_tree, geo["vstack"], "VS") if which == "V" else (bct.row_tree, geo["ustack"], "US")
    nodes = tree.nodes
    rank = (geo["rank_c"] if which == "V" else geo["rank_r"])[c]
    out = np.zeros((nodes[c].size, rank), dtype=np.complex128)
    for leaf, (W, cols) in stacks.items():
        L = nodes[leaf]
        if not (nodes[c].lo <= L.lo and L.hi <= nodes[c].hi):
            continue
        c0 = dict(cols)[c]
        blk = packed_arena[geo["offs"][(key, leaf)] : geo["offs"][(key, leaf)] + L.size * W].reshape(L.size, W)
        out[L.lo - nodes[c].lo : L.hi - nodes[c].lo] = blk[:, c0 : c0 + rank]
    return out


def _ancestors_in(tree, leaves, span, cset):
    """For every leaf position: the clusters of ``cset`` that contain it (root to leaf)."""
    anc = [[] for _ in leaves]
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


def pack(
    u,
    *,
    rows_per_chunk: int | None = None,
    near_interleave=None,
    near_interleave_adj=(0.4, 0.15, 0.3, 0.15),
    rank: int = 0,
    world: int = 1,
    stage_elems: int | None = None,
    peer: bool = False,
    factor_bias: float | None = None,
) -> PackedOperator:
    """Pack a UniformHMatrix (reference object or mirror) into arena + programs.

    ``world > 1``: the programs of one rank of the row-cluster partition.
    Output leaves are cut into ``world`` contiguous slices (``partition_bounds``); this rank
    runs P1/RED/U for the input clusters it owns (first index inside its input slice),
    NEAR/FAR for its output rows and Z for every output cluster touching its rows.  y/u live
    in an exchange region of the work buffer, one block per rank padded to ``ex_len``, filled
    for everyone by one in-place all-gather between launch A (P1, RED, U, NEAR) and launch B
    (Z, NEAR, FAR).

    ``peer=True`` (world > 1): ONE program per rank and direction instead of the A / B pair.
    The producers of this rank's y/u (P1 of single-chunk clusters, RED, U) also store them into
    every peer's exchange region (RUN_PEER) and signal their counters on every rank (OP_PEER);
    Z ops wait on remote counters with the owner's producer count.  The exchange rides the
    NVLink peer mappings inside the one kernel (csrc/uhmv_bulk.cuh, PEER)."""
    import os

    if rows_per_chunk is None:
        rows_per_chunk = int(os.environ.get("UHMV_ROWS_PER_CHUNK", ROWS_PER_CHUNK))
    if stage_elems is None:
        stage_elems = int(os.environ.get("UHMV_STAGE_ELEMS", STAGE_ELEMS))
    bct = u.bct
    n_rows, n_cols = bct.shape
    rnodes, cnodes = bct.row_tree.nodes, bct.col_tree.nodes

    # ---- which blocks / clusters take part (exactly what the reference walks) ----
    adm = []
    for s in bct.row_map:
        for t in bct.row_map[s]:
            adm.append((bct.block_of[(s, t)], s, t))
    rank_r = {s: int(u.row_basis.matrices[s].shape[1]) for s in bct.row_map}
    rank_c = {t: int(u.col_basis.matrices[t].shape[1]) for t in bct.col_map}
    if factor_bias is None:
        # operators under ~1 GB are bound by the forward dependency chain: product
        # form for every block whose factors are not at most half its size drops the U phase of
        # most blocks for ~2 % more streamed bytes (config 2 forward 0.61 -> 0.645; its adjoint,
        # which then sums more product-block partials, 0.56 -> 0.52)
        approx = sum(min(int(u.coeffs[bid].s_x.shape[1]) * (rank_r[s] + rank_c[t]), rank_r[s] * rank_c[t]) for bid, s, t in adm)
        approx += sum(int(np.prod(d.shape)) for d in u.dense.values())
        approx += sum(cnodes[t].size * rank_c[t] for t in bct.col_map) + sum(rnodes[s].size * rank_r[s] for s in bct.row_map)
        factor_bias = float(os.environ.get("UHMV_FACTOR_BIAS", FACTOR_BIAS_SMALL if 16 * approx < 1e9 else FACTOR_BIAS))
    adj_copy = world == 1 and os.environ.get("UHMV_ADJ_COPY", "1") != "0"
    kb, factorized = {}, {}
    bytes_coupling = 0
    for bid, s, t in adm:
        k = int(u.coeffs[bid].s_x.shape[1])
        kb[bid] = k
        ls, lt = rank_r[s], rank_c[t]
        factorized[bid] = k * (ls + lt) < factor_bias * ls * lt
        bytes_coupling += min(k * (ls + lt), ls * lt)  # the algorithmic bytes keep the min form
    dense_ids = list(u.dense.keys())

    # ---- arena layout ----
    offs = {}
    cursor = 0

    def alloc(key, n, ld):
        # every matrix starts at a multiple of its leading dimension: the multi-RHS engine
        # reads the arena as one 2-D TMA tensor per ld, (row, col) = divmod(offset, ld)
        nonlocal cursor
        if ld > 1:
            cursor = (cursor + ld - 1) // ld * ld
        offs[key] = cursor
        cursor += _align(max(n, 0))

    # Cluster bases are stored LEAF-STACKED: for every leaf L, the rows of the bases of all its
    # ancestors (root to leaf) side by side, [B_t1[L rows] | B_t2[L rows] | ...], one |L| x W_L
    # row-major matrix.  P1 (H) and FAR (N) of a leaf chunk then read ONE contiguous matrix
    # with W_L-long rows instead of one short-row slab per ancestor.
    vstack = _stacks(bct.col_tree, bct.col_map, rank_c)
    ustack = _stacks(bct.row_tree, bct.row_map, rank_r)
    for leaf, (W, _cols) in sorted(vstack.items()):
        alloc(("VS", leaf), cnodes[leaf].size * W, W)
    for leaf, (W, _cols) in sorted(ustack.items()):
        alloc(("US", leaf), rnodes[leaf].size * W, W)
    fcols = {}  # s -> ([(bid, t, pos, k)], kfac)
    spos, cwidth = {}, {}  # product block -> column in C_s; s -> width of C_s
    for s in sorted(bct.row_map):
        pos, cols = 0, []
        for t in bct.row_map[s]:
            bid = bct.block_of[(s, t)]
            if factorized[bid]:
                cols.append((bid, t, pos, kb[bid]))
                pos += kb[bid]
        fcols[s] = (cols, pos)
        # C_s = [F_s | S_b1 | S_b2 | ...]: the coupling of row cluster s as ONE l_s-row matrix
        # (factorized s_x columns, then the product-form blocks in row_map order), so the
        # forward Z op is a single long-row GEMV over all its inputs [u_b..., y_t...]
        w = pos
        for t in bct.row_map[s]:
            bid = bct.block_of[(s, t)]
            if not factorized[bid] and rank_c[t] > 0:
                spos[bid] = w
                w += rank_c[t]
        cwidth[s] = w
        alloc(("C", s), rank_r[s] * w, w)
        offs[("F", s)] = offs[("C", s)]
        for t in bct.row_map[s]:
            bid = bct.block_of[(s, t)]
            if bid in spos:
                offs[("S", bid)] = offs[("C", s)] + spos[bid]
    ycols = {}  # t -> ([(bid, s, pos, k)], K')
    for t in sorted(bct.col_map):
        pos, cols = 0, []
        for s in bct.col_map[t]:
            bid = bct.block_of[(s, t)]
            if factorized[bid]:
                cols.append((bid, s, pos, kb[bid]))
                pos += kb[bid]
        ycols[t] = (cols, pos)
        alloc(("Y", t), rank_c[t] * pos, pos)
    # Adjoint copy (single-GPU packs; UHMV_ADJ_COPY=0 turns it off): CT_t = [S_b^H ...] over the
    # product blocks of column cluster t, l_t rows, so the adjoint Z op of t is ONE long-row GEMV
    # over [y'_s ...] like the forward one over C_s -- no adjoint U ops and partial sums for
    # those blocks (a four-phase adjoint chain too).  Each direction streams its own copy: the
    # bytes per matvec do not change, the arena grows by the product-form coupling.
    ctpos, ctwidth = {}, {}
    if adj_copy:
        for t in sorted(bct.col_map):
            w = 0
            for s in bct.col_map[t]:
                bid = bct.block_of[(s, t)]
                if not factorized[bid] and rank_r[s] > 0 and rank_c[t] > 0:
                    ctpos[bid] = w
                    w += rank_r[s]
            if w:
                ctwidth[t] = w
                alloc(("CT", t), rank_c[t] * w, w)
    dense_by_rleaf, dense_by_cleaf = {}, {}
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
            alloc(("D", bid), rr * cc, cc)

    arena = np.zeros(max(cursor, ALIGN), dtype=np.complex128)

    def put(key, mat):
        m = np.asarray(mat)
        if m.size:
            arena[offs[key] : offs[key] + m.size] = m.reshape(-1)

    for key, stacks, nodes, basis in (("VS", vstack, cnodes, u.col_basis), ("US", ustack, rnodes, u.row_basis)):
        for leaf, (W, cols) in stacks.items():
            L = nodes[leaf]
            blk = arena[offs[(key, leaf)] : offs[(key, leaf)] + L.size * W].reshape(L.size, W)
            for c, c0 in cols:
                m = np.asarray(basis.matrices[c])
                blk[:, c0 : c0 + m.shape[1]] = m[L.lo - nodes[c].lo : L.hi - nodes[c].lo]
    for s, (cols, kfac) in fcols.items():
        ls, w = rank_r[s], cwidth[s]
        if ls and w:
            cs = np.empty((ls, w), dtype=np.complex128)
            for bid, t, pos, k in cols:
                cs[:, pos : pos + k] = u.coeffs[bid].s_x
            for t in bct.row_map[s]:
                bid = bct.block_of[(s, t)]
                if bid in spos:
                    pair = u.coeffs[bid]
                    cs[:, spos[bid] : spos[bid] + rank_c[t]] = pair.s_x @ np.conj(pair.s_y).T
            put(("C", s), cs)
    for t, w in ctwidth.items():
        ct = np.empty((rank_c[t], w), dtype=np.complex128)
        for s in bct.col_map[t]:
            bid = bct.block_of[(s, t)]
            if bid in ctpos:
                pair = u.coeffs[bid]
                ct[:, ctpos[bid] : ctpos[bid] + rank_r[s]] = np.conj(pair.s_x @ np.conj(pair.s_y).T).T
        put(("CT", t), ct)
    for t, (cols, ktot) in ycols.items():
        lt = rank_c[t]
        if lt and ktot:
            ys = np.empty((lt, ktot), dtype=np.complex128)
            for bid, s, pos, k in cols:
                ys[:, pos : pos + k] = u.coeffs[bid].s_y
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
        bct=bct, rank_r=rank_r, rank_c=rank_c, kb=kb, factorized=factorized,
        fcols=fcols, ycols=ycols, offs=offs, dense_by_rleaf=dense_by_rleaf, dense_by_cleaf=dense_by_cleaf,
        vstack=vstack, ustack=ustack, cwidth=cwidth, spos=spos, ctpos=ctpos, ctwidth=ctwidth,
    )
    if world > 1:
        part = _partition(geo, world, rank)
    else:
        part = None
    op_bytes = 16 * (bytes_bases + bytes_coupling + bytes_dense)
    tiny = op_bytes < 2e8  # config 1 (99 MB): bound by the P1 -> RED -> Z -> FAR chain
    if near_interleave is None:
        # forward nearfield shares between the farfield phases (measured): operators under
        # ~1 GB are chain-latency-bound and want the chain started early (configs 1-2: -3..4%);
        # under ~200 MB (product-form coupling: no U phase, so no share before Z) the nearfield
        # is split evenly around the chain (config 1: 0.302 -> 0.329,
        # profiles/r02b/sweep_near_shares_product_form.txt)
        small = op_bytes < 1e9
        near_interleave = (0.4, 0.2, 0.0, 0.4) if tiny else (0.2, 0.1, 0.2, 0.5) if small else (0.35, 0.1, 0.2, 0.35)
    if adj_copy and near_interleave_adj == (0.4, 0.15, 0.3, 0.15):
        # with the adjoint copy the adjoint chain mirrors the forward one (no U op or partial for
        # the product blocks) and wants the forward shares: config 2 adjoint 0.600 -> 0.627,
        # config 3 adjoint 0.913 -> 0.948 (profiles/r02b/ab_adjoint_copy{,_large}.txt)
        near_interleave_adj = (0.2, 0.1, 0.2, 0.5) if op_bytes < 1e9 else (0.35, 0.1, 0.2, 0.35)
    split_def = dict(SPLIT_DEFAULTS, **({"z_rows": 13} if tiny else {}))  # config 1: Z ops in two row parts
    split = {k: int(os.environ.get(f"UHMV_SPLIT_{k.upper()}", v)) for k, v in split_def.items()}
    if os.environ.get("UHMV_NEAR_INTERLEAVE"):
        near_interleave = tuple(float(v) for v in os.environ["UHMV_NEAR_INTERLEAVE"].split(","))
    if os.environ.get("UHMV_NEAR_INTERLEAVE_ADJ"):
        near_interleave_adj = tuple(float(v) for v in os.environ["UHMV_NEAR_INTERLEAVE_ADJ"].split(","))
    split["far_rows"] = int(os.environ.get("UHMV_FAR_ROWS", FAR_ROWS))
    split["z_elems"] = int(os.environ.get("UHMV_Z_ELEMS", 1 << 60))
    split["u_elems"] = int(os.environ.get("UHMV_U_ELEMS", 1 << 60))
    kw = dict(rows_per_chunk=rows_per_chunk, near_interleave=near_interleave, part=part, stage_elems=stage_elems,
              split=split, peer=bool(peer and world > 1), near_interleave_adj=near_interleave_adj,
              w_order=world == 1 and os.environ.get("UHMV_W_ORDER", "0") != "0")
    fwd, work_f, ex_f = _build_program(geo, adjoint=False, **kw)
    adj, work_a, ex_a = _build_program(geo, adjoint=True, **kw)
    _assign_tmaps([fwd, adj] + [q.part_b for q in (fwd, adj) if q.part_b is not None])
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
        rank=rank,
        world=world,
        part=part,
        exchange={"fwd": ex_f, "adj": ex_a},
        geo=geo,
        build_kw=kw,
        storage=dict(
            bases=16 * bytes_bases,
            coupling=16 * bytes_coupling,
            dense=16 * bytes_dense,
            # stored beyond §8d's minimum: the product-biased forms and the adjoint copy CT_t
            form_extra=16 * int(sum((kb[bid] * (rank_r[s] + rank_c[t]) if factorized[bid] else rank_r[s] * rank_c[t])
                                    for bid, s, t in adm) - bytes_coupling),
            adjoint_copy=16 * int(sum(rank_c[t] * w for t, w in ctwidth.items())),
            n_factorized=int(sum(factorized.values())),
            n_product=int(len(adm) - sum(factorized.values())),
        ),
    )


def partition_bounds(tree, world: int, weights=None, keep=()):
    """Cut the tree's index range into ``world`` contiguous slices on leaf boundaries.

    ``weights`` (leaf id -> bytes a rank streams for that leaf, :func:`leaf_bytes`): cut the
    prefix sums of the weights at r/world of the total -- row clusters partitioned by bytes
    touched (BASELINE north_star) -- only at leaf ends that cut no cluster of ``keep`` (a cut
    cluster's Z op would run on both ranks), when there are enough of those.  Without weights:
    leaf-balanced by index count."""
    leaves, _ = _leaves_under(tree)
    nodes = tree.nodes
    lo = nodes[getattr(tree, "root", 0)].lo
    hi = nodes[getattr(tree, "root", 0)].hi
    ends = [nodes[l].hi for l in leaves]
    if weights is not None and world > 1:
        cum = np.cumsum([float(weights.get(l, 0.0)) for l in leaves])
        total = float(cum[-1]) if len(cum) else 0.0
        if total > 0:
            kept = [nodes[c] for c in keep]
            ok = [i for i, e in enumerate(ends) if e < hi and not any(c.lo < e < c.hi for c in kept)]
            if len(ok) < world - 1:
                ok = [i for i, e in enumerate(ends) if e < hi]
            bounds = [lo]
            for r in range(1, world):
                target = total * r / world
                cand = [i for i in ok if ends[i] > bounds[-1]]
                if not cand:
                    bounds.append(hi)
                    continue
                best = min(cand, key=lambda i: abs(cum[i] - target))
                bounds.append(ends[best])
            bounds.append(hi)
            return bounds
    bounds = [lo]
    for r in range(1, world):
        target = lo + (hi - lo) * r / world
        # leaf end closest to the target, strictly after the previous cut
        best = min((e for e in ends if e > bounds[-1]), key=lambda e: abs(e - target), default=hi)
        bounds.append(best)
    bounds.append(hi)
    return bounds


def leaf_bytes(geo) -> dict:
    """Bytes one rank streams per row-tree leaf L of a forward matvec if it owns L (shared
    row / column tree): the dense blocks of L's rows (NEAR), L's row of the leaf stacks US_L
    and VS_L (FAR, P1), and the coupling C_s / Y_t of the clusters whose first leaf is L (Z,
    U).  None for two-tree operators (partition_bounds then cuts by index count)."""
    bct = geo["bct"]
    if bct.col_tree is not bct.row_tree:
        return None
    nodes = bct.row_tree.nodes
    leaves, span = _leaves_under(bct.row_tree)
    w = {l: 0 for l in leaves}
    for key, stacks in (("US", geo["ustack"]), ("VS", geo["vstack"])):
        for leaf, (W, _cols) in stacks.items():
            w[leaf] += nodes[leaf].size * W
    for leaf, bids in geo["dense_by_rleaf"].items():
        for bid in bids:
            r, c = bct.block_shape(bid)
            w[leaf] += r * c
    for s, wd in geo["cwidth"].items():
        w[leaves[span[s][0]]] += geo["rank_r"][s] * wd
    for t, (_cols, k) in geo["ycols"].items():
        w[leaves[span[t][0]]] += geo["rank_c"][t] * k
    return {l: 16 * v for l, v in w.items()}


def _partition(geo, world, rank):
    bct = geo["bct"]
    keep = [c for c in bct.row_map if geo["rank_r"][c] > 0]
    if bct.col_tree is bct.row_tree:
        keep += [c for c in bct.col_map if geo["rank_c"][c] > 0 and c not in bct.row_map]
    lb = leaf_bytes(geo)
    rb = partition_bounds(bct.row_tree, world, weights=lb, keep=keep)
    cb = rb if bct.col_tree is bct.row_tree else partition_bounds(bct.col_tree, world)
    return dict(rank=rank, world=world, row_bounds=rb, col_bounds=cb)


def _seg(m_off, buf, rows, cols, ld, mode, in_off, out_off, x_off=-1):
    """Logical segment; ``x_off`` >= 0 means the input vector is x[x_off : ...] (read in place
    by the bulk kernel, staged into xin at ``in_off`` by the register kernel)."""
    return (int(m_off), int(buf), int(rows), int(cols), int(ld), int(mode), int(in_off), int(out_off), int(x_off))


def _build_program(
    geo, *, adjoint: bool, rows_per_chunk: int, near_interleave, part=None, stage_elems=STAGE_ELEMS, split=None,
    peer=False, host_io=False, near_interleave_adj=None, w_order=False,
):
    """Returns (program, work length, exchange layout).  ``host_io``: the single-GPU variant
    whose P1 ops read x from the caller's pinned host buffer (and publish it to device x for
    the NEAR ops, which wait for it) and whose NEAR / FAR ops drain finished output leaves
    to the host buffer; (None, ...) when some input leaf has no P1 op or some output leaf
    no NEAR / FAR op (the caller then copies x and w around a plain launch)."""
    split = dict(SPLIT_DEFAULTS, **(split or {}))
    peer = bool(peer and part is not None)
    host_io = bool(host_io and part is None)
    if adjoint and near_interleave_adj is not None:
        near_interleave = near_interleave_adj
    bct = geo["bct"]
    offs = geo["offs"]
    fcols, ycols = geo["fcols"], geo["ycols"]
    factorized = geo["factorized"]
    if adjoint:
        in_tree, out_tree = bct.row_tree, bct.col_tree
        in_map, out_map = bct.row_map, bct.col_map
        in_rank, out_rank = geo["rank_r"], geo["rank_c"]
        in_stack_key, out_stack_key = "US", "VS"
        in_stacks, out_stacks = geo["ustack"], geo["vstack"]
        dense_by_outleaf = geo["dense_by_cleaf"]
    else:
        in_tree, out_tree = bct.col_tree, bct.row_tree
        in_map, out_map = bct.col_map, bct.row_map
        in_rank, out_rank = geo["rank_c"], geo["rank_r"]
        in_stack_key, out_stack_key = "VS", "US"
        in_stacks, out_stacks = geo["vstack"], geo["ustack"]
        dense_by_outleaf = geo["dense_by_rleaf"]
    in_nodes, out_nodes = in_tree.nodes, out_tree.nodes
    if part is not None:
        rank, world = part["rank"], part["world"]
        in_b = part["row_bounds"] if adjoint else part["col_bounds"]
        out_b = part["col_bounds"] if adjoint else part["row_bounds"]
        out_lo, out_hi = out_b[rank], out_b[rank + 1]

        def owner_in(t):
            lo = in_nodes[t].lo
            for r in range(world):
                if in_b[r] <= lo < in_b[r + 1]:
                    return r
            return world - 1

        def out_needed(s_):
            n_ = out_nodes[s_]
            return n_.lo < out_hi and n_.hi > out_lo
    else:
        rank, world = 0, 1
        out_lo, out_hi = 0, out_tree.nodes[getattr(out_tree, "root", 0)].hi

        def owner_in(t):
            return 0

        def out_needed(s_):
            return True

    def stack_segs(key, stacks, leaf, leaf_lo, a, b, clist, rank_of, mode, x_off):
        """Segments reading the basis rows [a, b) of clusters ``clist`` (root to leaf) from the
        leaf stack: ONE segment when they are adjacent columns of it (always at a single GPU;
        a rank's own clusters are the deep end of the chain), else one per cluster."""
        W, cols = stacks[leaf]
        c0 = dict(cols)
        base = offs[(key, leaf)] + (a - leaf_lo) * W
        first = c0[clist[0]]
        adjacent = all(c0[c] == first + sum(rank_of[q] for q in clist[:i]) for i, c in enumerate(clist))
        width = sum(rank_of[c] for c in clist)
        if adjacent:
            return [_seg(base + first, BUF_ARENA, b - a, width, W, mode, 0, 0, x_off)]
        out, o = [], 0
        for c in clist:
            r = rank_of[c]
            if mode == MODE_H:
                out.append(_seg(base + c0[c], BUF_ARENA, b - a, r, W, mode, 0, o, x_off))
            else:
                out.append(_seg(base + c0[c], BUF_ARENA, b - a, r, W, mode, o, 0, x_off))
            o += r
        return out

    # ---- work-buffer layout ----
    work = 0

    def walloc(n):
        nonlocal work
        o = work
        work += max(int(n), 0)
        return o

    in_leaves, in_span = _leaves_under(in_tree)
    out_leaves, out_span = _leaves_under(out_tree)
    in_anc = _ancestors_in(in_tree, in_leaves, in_span, [t for t in in_map if in_rank[t] > 0 and owner_in(t) == rank])
    out_anc = _ancestors_in(out_tree, out_leaves, out_span, [s for s in out_map if out_rank[s] > 0])

    p1_items = []  # (leafpos, lo, hi): every in-leaf split in <= P1_CHUNK rows
    for p, leaf in enumerate(in_leaves):
        if not in_anc[p]:
            continue
        n = in_nodes[leaf]
        for a, b in _chunks(n.lo, n.hi, P1_CHUNK):
            p1_items.append((p, a, b))
    if host_io and {q for q, _a, _b in p1_items} != set(range(len(in_leaves))):
        return None, 0, (0, 0)
    chunks_of = {t: [] for t in in_map}
    for idx, (p, a, b) in enumerate(p1_items):
        for t in in_anc[p]:
            chunks_of[t].append(idx)
    # exchange region: per owner rank, its input clusters' [y_t | u_t] in position order, every
    # rank block padded to the same length (in-place all-gather target)
    # u_t: forward, Y_t^H y_t (s_y of the factorized blocks); adjoint, u'_b = s_x^H y_s of the
    # factorized blocks of row cluster s.  The adjoint U op of s runs over its whole coupling
    # matrix C_s (packer arena) and also produces the partials S_b^H y_s of its product blocks,
    # stored per output cluster t and producing rank, contiguous, summed by t's Z op.
    u_len = {t: (ycols[t][1] if not adjoint else fcols[t][1]) for t in in_map}
    zparts = {}  # adjoint: (t, rank q) -> [product blocks (r, t) with owner_in(r) == q]
    use_ct = adjoint and world == 1 and bool(geo.get("ctwidth"))  # adjoint copy CT_t: no partials
    if adjoint and not use_ct:
        for t in sorted(out_map, key=lambda t: out_nodes[t].lo):
            if out_rank[t] == 0:
                continue
            for r in out_map[t]:
                bid = bct.block_of[(r, t)]
                if not factorized[bid] and in_rank[r] > 0:
                    zparts.setdefault((t, owner_in(r)), []).append(bid)
    by_rank = [[] for _ in range(world)]
    for t in sorted(in_map, key=lambda t: in_nodes[t].lo):
        by_rank[owner_in(t)].append(t)
    zp_len = [0] * world
    for (t, q), bids in zparts.items():
        zp_len[q] += len(bids) * out_rank[t]
    ex_len = max([sum(in_rank[t] + u_len[t] for t in ts) + zp_len[r] for r, ts in enumerate(by_rank)] + [0])
    y_off, u_off, zp_off = {}, {}, {}
    for r, ts in enumerate(by_rank):
        cur = r * ex_len
        for t in ts:
            y_off[t] = cur
            cur += in_rank[t]
            u_off[t] = cur
            cur += u_len[t]
        for (t, q), bids in sorted(zparts.items(), key=lambda kv: (out_nodes[kv[0][0]].lo, kv[0][1])):
            if q == r:
                zp_off[(t, q)] = cur
                cur += len(bids) * out_rank[t]
    zp_slot = {}  # product block -> its partial's work offset
    for (t, q), bids in zparts.items():
        for i, bid in enumerate(bids):
            zp_slot[bid] = zp_off[(t, q)] + i * out_rank[t]
    walloc(world * ex_len)
    part_off = {}
    for t in sorted(in_map, key=lambda t: in_nodes[t].lo):
        if in_rank[t] and owner_in(t) == rank:
            part_off[t] = y_off[t] if len(chunks_of[t]) == 1 else walloc(len(chunks_of[t]) * in_rank[t])
    z_off = {}
    for s in sorted(out_map, key=lambda s: out_nodes[s].lo):
        z_off[s] = walloc(out_rank[s])
    u_pos = {}
    for t in in_map:
        for entry in (ycols[t][0] if not adjoint else fcols[t][0]):
            u_pos[entry[0]] = entry[2]

    # ---- dependency counters ----
    n_ctr = 0

    def ctr():
        nonlocal n_ctr
        n_ctr += 1
        return n_ctr - 1

    c_part = {t: ctr() for t in in_map}
    c_y = {t: ctr() for t in in_map}
    c_u = {t: ctr() for t in in_map}
    c_z = {s: ctr() for s in out_map}
    in_pos = {leaf: q for q, leaf in enumerate(in_leaves)}
    c_x = {q: ctr() for q in range(len(in_leaves))} if host_io else {}  # x[leaf] is in device x
    c_w = {q: ctr() for q in range(len(out_leaves))} if host_io else {}  # contributions to w[leaf]
    ops = {k: [] for k in range(7)}

    # P1: partial_t = B_t[chunk rows]^H x[chunk]; the ancestors of a chunk are grouped into
    # ops of <= split["p1_out"] outputs so the head of the dependency chain spreads over CTAs
    for idx, (p, a, b) in enumerate(p1_items):
        groups, cur, tot = [], [], 0
        for t in in_anc[p]:
            if cur and tot + in_rank[t] > split["p1_out"]:
                groups.append(cur)
                cur, tot = [], 0
            cur.append(t)
            tot += in_rank[t]
        if cur:
            groups.append(cur)
        leaf = in_leaves[p]
        for grp in groups:
            segs, outs, sigs = [], [], []
            oo = 0
            for t in grp:
                lt = in_rank[t]
                outs.append((BUF_WORK, part_off[t] + chunks_of[t].index(idx) * lt, lt, oo, 0))
                sigs.append(c_part[t])
                oo += lt
            segs = stack_segs(in_stack_key, in_stacks, leaf, in_nodes[leaf].lo, a, b, grp, in_rank, MODE_H,
                              -1 if host_io else a)
            kind = KIND_P1
            if host_io:  # x[a:b] gathered from the host, published to device x
                kind |= OP_XHOST
                sigs.append(c_x[p])
            ops[KIND_P1].append((kind, b - a, oo, [(BUF_X, a, b - a, 0, 0)], segs, outs, [], sigs, (b - a) * oo))
    # RED: y_t = sum of chunk partials (skipped when the single partial is y_t itself)
    for t in in_map:
        lt, nchunk = in_rank[t], len(chunks_of[t])
        if lt == 0 or nchunk <= 1 or owner_in(t) != rank:
            continue
        segs = [_seg(part_off[t], BUF_WORK, nchunk, lt, lt, MODE_S, 0, 0)]
        ops[KIND_RED].append(
            (KIND_RED, 0, lt, [], segs, [(BUF_WORK, y_off[t], lt, 0, 0)], [(c_part[t], nchunk)], [c_y[t]], nchunk * lt)
        )
    # peer exchange: waits on counters another rank signals carry that owner's producer
    # count (every rank derives it from the same structure: P1 chunks under t, U panels)
    remote_ctr = set()
    n_chunks_all = {}
    if peer:
        for t in in_map:
            a_, b_ = in_span[t]
            n_chunks_all[t] = sum(
                len(_chunks(in_nodes[in_leaves[q]].lo, in_nodes[in_leaves[q]].hi, P1_CHUNK)) for q in range(a_, b_)
            )
            if owner_in(t) == rank and in_rank[t]:
                assert n_chunks_all[t] == len(chunks_of[t])
    y_wait = {}
    for t in in_map:
        if in_rank[t] and owner_in(t) != rank and peer:
            y_wait[t] = [(c_part[t], 1)] if n_chunks_all[t] <= 1 else [(c_y[t], 1)]
            remote_ctr.add(y_wait[t][0][0])
        elif in_rank[t] == 0 or owner_in(t) != rank:
            y_wait[t] = []  # zero-width, or produced by another rank (ordered by the exchange)
        elif len(chunks_of[t]) <= 1:
            y_wait[t] = [(c_part[t], len(chunks_of[t]))]
        else:
            y_wait[t] = [(c_y[t], 1)]
    # U: staging vectors of the factorized blocks.  l_t = 0 gives exact zeros (reference:
    # (k x 0) @ (0,)), which the zero-initialised, never-written work region already holds.
    def u_panel_step(lt, n):
        """Columns per U op: split["u_cols"], or equal panels (multiples of 8) of at most
        split["u_elems"] matrix elements -- long U ops delay every Z op behind them."""
        step = split["u_cols"]
        if lt * n > split.get("u_elems", 1 << 60):
            step = min(step, (-(-n // -(-(lt * n) // split["u_elems"])) + 7) // 8 * 8)
        return max(step, 8)

    u_wait = {}
    for t in in_map:
        n, lt = u_len[t], in_rank[t]
        u_wait[t] = []
        if (n == 0 and not (adjoint and not use_ct and geo["cwidth"][t])) or lt == 0:
            continue
        if owner_in(t) != rank:
            if peer:  # the owner's U panels of t, signalled across ranks
                n_u = geo["cwidth"][t] if adjoint else n
                u_wait[t] = [(c_u[t], len(_chunks(0, n_u, u_panel_step(lt, n_u))))]
                remote_ctr.add(c_u[t])
            continue
        u_wait[t] = [(c_u[t], 1)]
        if not adjoint:
            base, ld, outs = offs[("Y", t)], n, [(BUF_WORK, u_off[t], n, 0, 0)]
        elif use_ct:  # adjoint copy: only F_s -> [u'_b ...]; the product blocks go through CT_t in the Z ops
            base, ld, outs = offs[("C", t)], geo["cwidth"][t], [(BUF_WORK, u_off[t], n, 0, 0)]
        else:  # the whole C_s: [F_s | S_b ...] -> [u'_b ... | partial slots of the product blocks]
            base, ld = offs[("C", t)], geo["cwidth"][t]
            outs = [(BUF_WORK, u_off[t], n, 0, 0)] if n else []
            for r2 in bct.row_map[t]:
                bid = bct.block_of[(t, r2)]
                if bid in zp_slot:
                    outs.append((BUF_WORK, zp_slot[bid], out_rank[r2], geo["spos"][bid], 0))
            n = ld
        for c0, c1 in _chunks(0, n, u_panel_step(lt, n)):  # column panels: one op each
            segs = [_seg(base + c0, BUF_ARENA, lt, c1 - c0, ld, MODE_H, 0, 0)]
            ops[KIND_U].append(
                (KIND_U, lt, c1 - c0, [(BUF_WORK, y_off[t], lt, 0, 0)], segs, _clip_runs(outs, c0, c1),
                 list(y_wait[t]), [c_u[t]], lt * (c1 - c0))
            )
    # Z: coupling, owned by the output cluster (row cluster forward, column cluster adjoint)
    for s in out_map:
        ls = out_rank[s]
        if ls == 0 or not out_needed(s):
            continue
        in_runs, segs, waits = [], [], []
        if not adjoint:
            cols, kfac = fcols[s]
            for bid, t, pos, k in cols:  # F_s [u_b ...]
                if k:
                    in_runs.append((BUF_WORK, u_off[t] + u_pos[bid], k, pos, 0))
                    waits.extend(u_wait[t])
            n_in = kfac
            for t in out_map[s]:  # + S_b y_t for product blocks (C_s columns after F_s)
                bid = bct.block_of[(s, t)]
                lt = in_rank[t]
                if factorized[bid] or lt == 0:
                    continue
                in_runs.append((BUF_WORK, y_off[t], lt, n_in, 0))
                waits.extend(y_wait[t])
                n_in += lt
            assert n_in == geo["cwidth"][s]
            if n_in:  # one segment: the whole C_s
                segs.append(_seg(offs[("C", s)], BUF_ARENA, ls, n_in, n_in, MODE_N, 0, 0))
            nbytes = ls * n_in
        else:
            cols, ktot = ycols[s]
            for bid, r, pos, k in cols:  # Y_t [u'_b ...]
                if k:
                    in_runs.append((BUF_WORK, u_off[r] + u_pos[bid], k, pos, 0))
                    waits.extend(u_wait[r])
            if ktot:
                segs.append(_seg(offs[("Y", s)], BUF_ARENA, ls, ktot, ktot, MODE_N, 0, 0))
            n_in = ktot
            nbytes = ls * ktot
            ctw = geo["ctwidth"].get(s, 0) if use_ct else 0
            if ctw:  # + CT_s [y'_r ...]: the product blocks of column cluster s in one long-row GEMV
                for r in bct.col_map[s]:
                    bid = bct.block_of[(r, s)]
                    if bid in geo["ctpos"]:
                        in_runs.append((BUF_WORK, y_off[r], in_rank[r], ktot + geo["ctpos"][bid], 0))
                        waits.extend(y_wait[r])
                segs.append(_seg(offs[("CT", s)], BUF_ARENA, ls, ctw, ctw, MODE_N, ktot, 0))
                n_in = ktot + ctw
                nbytes += ls * ctw
            for r in out_map[s]:  # + S_b^H y'_r of product blocks: computed by U_r ...
                bid = bct.block_of[(r, s)]
                if bid in zp_slot:
                    waits.extend(u_wait[r])
            for q in range(world):  # ... and summed here, one contiguous run per producing rank
                bids = zparts.get((s, q), [])
                if bids:
                    segs.append(_seg(zp_off[(s, q)], BUF_WORK, len(bids), ls, ls, MODE_S, 0, 0))
                    nbytes += len(bids) * ls
        z_step = split["z_rows"]
        if nbytes > split.get("z_elems", 1 << 60):  # long ops bound the Z phase: equal row parts
            z_step = min(z_step, -(-ls // -(-nbytes // split["z_elems"])))
        for o0, o1 in _chunks(0, ls, z_step):  # output-row parts: one op each
            part = _restrict(segs, o0, o1)
            nb = sum(q[2] * q[3] for q in part)
            ops[KIND_Z].append(
                (KIND_Z, n_in, o1 - o0, in_runs, part, [(BUF_WORK, z_off[s] + o0, o1 - o0, 0, 0)],
                 sorted(set(waits)), [c_z[s]], nb)
            )

    # NEAR + FAR per output-leaf chunk
    # The output w is zeroed by the launcher and every entry receives at most one NEAR and one
    # FAR contribution through fp64 atomic adds: with two addends onto zero the sum is
    # order-independent (fl(a+b) = fl(b+a)), so NEAR and FAR need no ordering between them.
    # Ordered output (``w_order``, single-GPU programs): the NEAR ops of a leaf STORE their rows
    # and signal the leaf's counter, its FAR ops wait for them and add with a plain
    # read-modify-write -- no zeroing pass over w, no atomics, a fixed order.  It needs every
    # output leaf to have a NEAR or a FAR op (else the launcher's memset + red.add scheme stays).
    if w_order and not host_io and world == 1:
        for p, leaf in enumerate(out_leaves):
            if not dense_by_outleaf.get(leaf, []) and not out_anc[p]:
                w_order = False
    else:
        w_order = False
    c_near = {}
    for p, leaf in enumerate(out_leaves):
        n = out_nodes[leaf]
        if not (out_lo <= n.lo and n.hi <= out_hi):
            continue  # another rank's output rows
        dlist = dense_by_outleaf.get(leaf, [])
        if w_order and dlist:
            c_near[p] = ctr()
        # forward: row chunks of the leaf; adjoint: the whole column leaf (H segments reduce
        # over the block rows, so the op owns all |c| output entries of the leaf)
        # (adjoint: column panels of the leaf, ADJ_NEAR_COLS wide -- the H segments reduce over
        # the block rows, so an op owns whole output columns)
        near_chunks = _chunks(n.lo, n.hi, rows_per_chunk if not adjoint else ADJ_NEAR_COLS)
        for a, b in near_chunks:
            if not dlist:
                continue
            rows = b - a
            in_runs, segs = [], []
            pos = 0
            nbytes = 0
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
                    segs.append(_seg(offs[("D", bid)] + (a - n.lo), BUF_ARENA, r.size, rows, n.size, MODE_H, pos, 0, r.lo))
                    pos += r.size
                    nbytes += r.size * rows
            kind, waits_n, outs_n = KIND_NEAR, [], [(BUF_W, a, rows, 0, 0 if w_order else RUN_ATOMIC)]
            if host_io:
                kind |= OP_XWAIT | OP_DRAIN
                leaves_in = sorted({in_pos[bct.nodes[bid].col if not adjoint else bct.nodes[bid].row] for bid in dlist})
                waits_n = [(c_x[q], 0) for q in leaves_in]
                outs_n.append((BUF_HOSTW, n.lo, n.size, c_w[p], 0))
            ops[KIND_NEAR].append((kind, pos, rows, in_runs, segs, outs_n, waits_n,
                                   [c_near[p]] if p in c_near else [], nbytes))
        anc = out_anc[p]
        if not anc:
            continue
        for a, b in _chunks(n.lo, n.hi, split["far_rows"]):
            rows = b - a
            in_runs, segs, waits = [], [], []
            pos = 0
            for s in anc:
                ls = out_rank[s]
                in_runs.append((BUF_WORK, z_off[s], ls, pos, 0))
                waits.append((c_z[s], 1))
                pos += ls
            segs = stack_segs(out_stack_key, out_stacks, leaf, n.lo, a, b, anc, out_rank, MODE_N, -1)
            kind, outs_f = KIND_FAR, [(BUF_W, a, rows, 0, RUN_ATOMIC)]
            if w_order:  # after the leaf's NEAR stores (or alone on the leaf: a store)
                outs_f = [(BUF_W, a, rows, 0, RUN_ADD if p in c_near else 0)]
                if p in c_near:
                    waits.append((c_near[p], 1))
            if host_io:
                kind |= OP_DRAIN
                outs_f.append((BUF_HOSTW, n.lo, n.size, c_w[p], 0))
            ops[KIND_FAR].append((kind, pos, rows, in_runs, segs, outs_f, waits, [], rows * pos))

    # ---- a wait means "every op signalling this counter is done": count the producers ----
    producers = {}
    for k in ops:
        for o in ops[k]:
            for c in o[7]:
                producers[c] = producers.get(c, 0) + 1
    for k in ops:
        ops[k] = [
            o[:6] + ([(c, producers.get(c, _n if c in remote_ctr else 0)) for c, _n in o[6]],) + o[7:]
            for o in ops[k]
        ]
    if host_io:  # every output leaf drains once: its NEAR + FAR op count is the drain target
        n_contrib = {}
        for k in (KIND_NEAR, KIND_FAR):
            for o in ops[k]:
                for r in o[5]:
                    if r[0] == BUF_HOSTW:
                        n_contrib[r[3]] = n_contrib.get(r[3], 0) + 1
        if set(n_contrib) != set(c_w.values()):
            return None, 0, (0, 0)
        for k in (KIND_NEAR, KIND_FAR):
            ops[k] = [
                o[:5] + ([r if r[0] != BUF_HOSTW else r[:4] + (n_contrib[r[3]],) for r in o[5]],) + o[6:]
                for o in ops[k]
            ]
    # ---- order: largest first inside each kind (reference uniform.py:505-506) ----
    for k in ops:
        ops[k].sort(key=lambda o: -o[-1])
    if host_io:
        # x arrives over PCIe through the P1 ops: run them in tree order, and the NEAR ops
        # (which wait for the x of their column leaves, mostly tree neighbours) likewise
        ops[KIND_P1].sort(key=lambda o: o[3][0][1])
        ops[KIND_NEAR].sort(key=lambda o: [r for r in o[5] if r[0] == BUF_W][0][1])
    near = ops[KIND_NEAR]
    f = np.cumsum([0.0] + list(near_interleave))
    f = f / f[-1]
    cut = [int(round(x * len(near))) for x in f]
    near_parts = [near[cut[i] : cut[i + 1]] for i in range(len(near_interleave))]
    while len(near_parts) < 4:
        near_parts.append([])
    if w_order:  # FAR ops wait for the NEAR ops of their leaf: no nearfield share behind them
        near_parts = near_parts[:3] + [[o for part in near_parts[3:] for o in part]]
    # phased launches (multi-launch mode): [P1 + NEAR] [RED] [U] [Z] [FAR]
    phased = [ops[KIND_P1] + near]
    phased += [ops[k] for k in (KIND_RED, KIND_U, KIND_Z, KIND_FAR)]
    ex = (0, ex_len)
    if world == 1 or peer:
        # fused persistent order: every op waits only on ops that come earlier; nearfield ops
        # (no dependencies) are spread between the dependent farfield phases to cover latency
        fused = (
            ops[KIND_P1] + near_parts[0] + ops[KIND_RED] + near_parts[1] + ops[KIND_U] + near_parts[2]
            + ops[KIND_Z] + near_parts[3] + ops[KIND_FAR] + [o for part in near_parts[4:] for o in part]
        )
        prog = _finish(phased, fused, n_ctr, stage_elems=stage_elems, peer_limit=world * ex_len if peer else None)
        prog.zero_output = not w_order
        prog.w_order = bool(w_order)
        return prog, work, ex
    # multi-GPU: launch A produces this rank's y/u (+ nearfield), the exchange fills every
    # rank's y/u, launch B consumes them.  Waits on ops outside a launch are dropped: they are
    # ordered by the launch boundary and the all-gather.
    a_ops = ops[KIND_P1] + near_parts[0] + ops[KIND_RED] + near_parts[1] + ops[KIND_U] + near_parts[2]
    b_ops = ops[KIND_Z] + near_parts[3] + ops[KIND_FAR]
    prog_a = _finish([a_ops], a_ops, n_ctr, stage_elems=stage_elems)
    prog_b = _finish([b_ops], b_ops, n_ctr, keep_waits_on=KIND_Z, stage_elems=stage_elems)
    prog_b.zero_output = False
    prog_a.part_b = prog_b
    return prog_a, work, ex


def _clip_runs(runs, c0, c1):
    """The output runs of vector positions [c0, c1), re-based to start at 0."""
    out = []
    for buf, off, ln, dst, fl in runs:
        a, b = max(dst, c0), min(dst + ln, c1)
        if a < b:
            out.append((buf, off + (a - dst), b - a, a - c0, fl))
    return out


def _restrict(segs, o0, o1):
    """The part of an op's logical segments that produces output entries [o0, o1) (N: rows,
    H/S: columns), re-based so the part's outputs start at 0."""
    out = []
    for m_off, buf, rows, cols, ld, mode, in_off, out_off, x_off in segs:
        span = rows if mode == MODE_N else cols
        lo, hi = max(o0, out_off), min(o1, out_off + span)
        if lo >= hi:
            continue
        d = lo - out_off
        if mode == MODE_N:
            out.append((m_off + d * ld, buf, hi - lo, cols, ld, mode, in_off, lo - o0, x_off))
        else:
            out.append((m_off + d, buf, rows, hi - lo, ld, mode, in_off, lo - o0, x_off))
    return out


def _panel_split(s):
    """Register-kernel form of a logical segment: H/S split in <= HCOLS_MAX columns."""
    m_off, buf, rows, cols, ld, mode, in_off, out_off, _x = s
    if mode == MODE_N or cols <= HCOLS_MAX:
        return [(m_off, buf, rows, cols, ld, mode, in_off, out_off)]
    return [(m_off + c0, buf, rows, c1 - c0, ld, mode, in_off, out_off + c0) for c0, c1 in _chunks(0, cols, HCOLS_MAX)]


def _order_segments(segs):
    """N segments first (grouped by out_off/rows), then H/S groups (by out_off/cols).

    Both kernels rely on it: N rows are owner-updated without a barrier, and one barrier
    at the N -> H switch orders them before the H owners touch the same outputs."""
    n = [s for s in segs if s[5] == MODE_N]
    h = [s for s in segs if s[5] != MODE_N]
    n.sort(key=lambda s: (s[7], s[2]))
    h.sort(key=lambda s: (s[5], s[7], s[3]))
    return n + h


def _pieces(segs, has_x, stage_elems=STAGE_ELEMS, ncols_max=BULK_NCOLS_MAX, h_panel=BULK_HCOLS_MAX):
    """Cut an op's logical segments into row ranges packed into STAGE_ELEMS stages.

    Pieces whose input is a window of x (P1 and NEAR ops) carry that window inside the stage,
    right behind their matrix rows (PI_XSTAGE): the producer bulk-copies it from x (L2-resident)
    so the consumers never gather x.  Their ``in_off`` is then the x index of the window."""
    out = []
    fill = 0  # elements used in the open stage
    open_idx = None  # index in ``out`` of the open stage's first piece

    def close():
        nonlocal fill, open_idx
        if open_idx is not None:
            out[-1][7] |= PI_END
            out[open_idx][7] |= fill << 32
        fill = 0
        open_idx = None

    split = []
    for sg in segs:  # H/S groups own at most BULK_HCOLS_MAX output columns: cut wider ones
        m_off, buf, rows, cols, ld, mode, in_off, out_off, x_off = sg[:9]
        alias = sg[9] if len(sg) > 9 else ()
        if mode != MODE_N and cols > min(h_panel, stage_elems // 2):
            for c0, c1 in _chunks(0, cols, min(h_panel, stage_elems // 2)):
                split.append((m_off + c0, buf, rows, c1 - c0, ld, mode, in_off, out_off + c0, x_off, ()))
        elif mode == MODE_N and cols > min(ncols_max, stage_elems // 2):  # rows wider than a stage
            for c0, c1 in _chunks(0, cols, min(ncols_max, stage_elems // 2)):  # -> column panels
                sub = []  # the alias sub-blocks (column ranges) that fall into this panel
                for a0, ac, amode, a_in, a_out in alias:
                    lo, hi = max(a0, c0), min(a0 + ac, c1)
                    if lo < hi:
                        sub.append((lo - c0, hi - lo, amode, a_in, a_out + (lo - a0)))
                split.append((m_off + c0, buf, rows, c1 - c0, ld, mode, in_off + c0, out_off,
                              x_off + c0 if x_off >= 0 else x_off, tuple(sub)))
        else:
            split.append(tuple(sg[:9]) + (alias,))
    for m_off, buf, rows, cols, ld, mode, in_off, out_off, x_off, alias in split:
        xs = x_off >= 0 and has_x
        if buf == BUF_WORK:  # coherent in-kernel data: no bulk copy, no stage
            close()  # the open stage ends with the last staged piece
            out.append([m_off, ld, rows, cols, mode, in_off, out_off, PI_DIRECT])
            continue
        # elements a piece of n rows occupies in a stage (matrix + its x window)
        per_row = cols + (1 if (xs and mode != MODE_N) else 0)
        extra = cols if (xs and mode == MODE_N) else 0
        if per_row + extra > stage_elems:
            raise ValueError(f"segment row of {cols} elements exceeds a {stage_elems}-element stage")
        r = 0
        # a narrow N segment that fits a whole stage is not cut at a stage boundary when the room
        # left is small: the cut costs two half-empty passes of the 16 row groups
        if (mode == MODE_N and NOSPLIT > 0 and fill > 0 and rows * per_row + extra <= stage_elems
                and fill + rows * per_row + extra > stage_elems
                and stage_elems - fill <= NOSPLIT * stage_elems):
            close()
        while r < rows:
            room = (stage_elems - fill - extra) // per_row
            if room <= 0:
                close()
                room = (stage_elems - extra) // per_row
            n = min(room, rows - r)
            info = fill | (PI_XSTAGE if xs else 0)
            if open_idx is None:
                info |= PI_BEGIN
                open_idx = len(out)
            if xs:
                in_v = x_off + (r if mode != MODE_N else 0)
            else:
                in_v = in_off + (r if mode != MODE_N else 0)
            out.append([m_off + r * ld, ld, n, cols, mode, in_v, out_off + (r if mode == MODE_N else 0), info])
            # alias pieces: the same staged rows used a second time (one HBM read, two products)
            for a0, ac, amode, a_in, a_out in alias:
                out.append([m_off + r * ld + a0, ld, n, ac, amode, a_in + r, a_out, (fill + a0) | PI_ALIAS | (cols << 32)])
            fill += n * per_row + extra
            r += n
    close()
    return out


def _resolve_inputs(segs, in_runs):
    """Multi-RHS form of an op's segments: each one reads its input from ONE contiguous
    source (x or work) at an absolute element index; a segment whose input window spans
    several gather runs (F_s over many u_b vectors) is cut at the run boundaries
    (column ranges for N, row ranges for H/S)."""
    runs = sorted(in_runs, key=lambda r: r[3])  # (buf, off, len, dst, flags) by xin position
    out = []
    for m_off, buf, rows, cols, ld, mode, in_off, out_off, _x in segs:
        if mode == MODE_S:
            out.append((m_off, ld, rows, cols, mode, -1, 0, out_off))
            continue
        span = cols if mode == MODE_N else rows
        pos = in_off
        end = in_off + span
        while pos < end:
            r = next(rr for rr in runs if rr[3] <= pos < rr[3] + rr[2])
            take = min(end, r[3] + r[2]) - pos
            k0 = pos - in_off
            src = r[1] + (pos - r[3])
            if mode == MODE_N:
                out.append((m_off + k0, ld, rows, take, mode, r[0], src, out_off))
            else:
                out.append((m_off + k0 * ld, ld, take, cols, mode, r[0], src, out_off))
            pos += take
    return out


def _assign_tmaps(progs):
    """Give every multi-RHS arena segment the index of its leading dimension in one sorted
    list shared by ``progs`` (mode-field bits 16..; the device plan encodes one pair of TMA
    tensor maps per distinct ld over the arena)."""
    lds = sorted({int(q[1]) for p in progs for q in p.mr_segs if (q[4] & 0xFF) != MODE_S})
    index = {ld: i for i, ld in enumerate(lds)}
    for p in progs:
        m = p.mr_segs.copy()
        for q in m:
            if (q[4] & 0xFF) != MODE_S:
                q[4] = (q[4] & 0xFFFF) | (index[int(q[1])] << MR_TMAP_SHIFT)
        p.mr_segs = m
        p.mr_lds = np.asarray(lds, dtype=np.int64)


def _mr_groups(mr, n_out):
    """Mark the group structure of an op's multi-RHS segments.  A group is a run of
    consecutive segments with the same mode and outputs (the engines accumulate it in
    registers and flush once); the first group writing an output range gets MR_FIRST (its
    flush stores).  Returns (segments, op flags): MR_ZERO when some output is left unwritten."""
    out = []
    covered = np.zeros(n_out, dtype=bool)
    i = 0
    while i < len(mr):
        mode, o = mr[i][4], mr[i][7]
        nout = mr[i][2] if mode == MODE_N else mr[i][3]
        j = i + 1
        while j < len(mr) and mr[j][4] == mode and mr[j][7] == o and (mr[j][2] if mode == MODE_N else mr[j][3]) == nout:
            j += 1
        first = not covered[o : o + nout].any()
        covered[o : o + nout] = True
        out.extend(q[:4] + (q[4] | (MR_FIRST if first else 0),) + q[5:] for q in mr[i:j])
        i = j
    return out, (0 if covered.all() else MR_ZERO)


def _finish(phased, fused, n_ctr, keep_waits_on=None, stage_elems=STAGE_ELEMS, peer_limit=None,
            h_panel=BULK_HCOLS_MAX, bulk_only=False):
    """Flatten op tuples into arrays in the phased order; the fused order is a
    permutation (``fused_order[ticket] = op index``).  ``keep_waits_on``: in a partial program
    keep only waits on counters signalled by ops of this kind inside the program.
    ``peer_limit``: peer-exchange program -- work outputs below this offset (the y/u exchange
    region) are RUN_PEER runs and their ops are flagged OP_PEER."""
    order = [o for ph in phased for o in ph]
    host_io = False
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
    segs, pieces, runs, waits, sigs = [], [], [], [], []
    mr_segs, mr_ranges = [], []
    in_max = xin_max = out_max = 0
    arena_elems = 0
    local_ctr = None
    if keep_waits_on is not None:
        local_ctr = {c for o in order if o[0] == keep_waits_on for c in o[7]}
    for i, (kind, n_in, n_out, in_runs, sg, out_runs, wt, sgn, _) in enumerate(order):
        if local_ctr is not None:
            wt = [w for w in wt if w[0] in local_ctr]
        arena_elems += sum(q[2] * q[3] for q in sg if q[1] == BUF_ARENA)
        has_x = any(r[0] == BUF_X for r in in_runs)
        has_w = any(r[0] == BUF_WORK for r in in_runs)
        assert not (has_x and has_w), "an op reads x or work inputs, never both"
        op_flags = 0
        if peer_limit is not None:
            marked = []
            for buf, off, ln, dst, fl in out_runs:
                if buf == BUF_WORK and off < peer_limit:
                    assert off + ln <= peer_limit and not fl & (RUN_ADD | RUN_ATOMIC)
                    fl |= RUN_PEER
                    op_flags = OP_PEER
                marked.append((buf, off, ln, dst, fl))
            out_runs = marked
        drain = [r for r in out_runs if r[0] == BUF_HOSTW]
        out_runs = [r for r in out_runs if r[0] != BUF_HOSTW]
        in_b = len(runs)
        runs.extend(in_runs)
        in_e = len(runs)
        out_b = len(runs)
        runs.extend(out_runs)
        out_e = len(runs)
        runs.extend(drain)  # read by OP_DRAIN ops at index out_e, outside the output cover
        host_io = host_io or bool(kind & (OP_XHOST | OP_XWAIT | OP_DRAIN))
        ordered = _order_segments(sg)
        seg_b = len(segs)
        for s in ordered:
            segs.extend(_panel_split(s[:9]))
        seg_e = len(segs)
        pc_b = len(pieces)
        nsg = [q for q in ordered if q[5] == MODE_N]
        wide = bool(nsg) and all(q[3] >= WIDE_COLS for q in nsg)
        # warp-per-row ops: panels narrow enough that a stage holds a row for every warp
        pcs = _pieces(ordered, has_x, stage_elems, NW_COLS if wide else BULK_NCOLS_MAX, h_panel)
        if wide:  # long rows: few per piece
            for pc in pcs:
                if pc[4] == MODE_N:
                    pc[4] = MODE_NW
        pieces.extend(pcs)
        pc_e = len(pieces)
        mr_b = len(mr_segs)
        mr, mr_flags = ([], 0) if bulk_only else _mr_groups(_resolve_inputs([q[:9] for q in ordered], in_runs), n_out)
        mr_segs.extend(mr)
        mr_ranges.append((mr_b, len(mr_segs), mr_flags))
        w_b = len(waits)
        waits.extend(wt)
        w_e = len(waits)
        s_b = len(sigs)
        sigs.extend(sgn)
        s_e = len(sigs)
        xin_len = 0 if (has_x and not kind & (OP_XHOST | OP_XIN)) else n_in  # x windows travel in the stages
        ops[i] = (n_in, n_out, in_b, in_e, seg_b, seg_e, out_b, out_e, w_b, w_e, s_b, s_e, kind | op_flags, pc_b, pc_e,
                  xin_len)
        in_max = max(in_max, n_in)
        xin_max = max(xin_max, xin_len)
        out_max = max(out_max, n_out)
    return Program(
        ops=ops,
        segs=np.asarray(segs, dtype=np.int64).reshape(-1, SEG_FIELDS),
        pieces=np.asarray(pieces, dtype=np.int64).reshape(-1, PIECE_FIELDS),
        runs=np.asarray(runs, dtype=np.int64).reshape(-1, RUN_FIELDS),
        waits=np.asarray(waits, dtype=np.int32).reshape(-1, 2),
        sigs=np.asarray(sigs, dtype=np.int32).reshape(-1),
        phases=bounds,
        fused_order=fused_order,
        in_max=in_max,
        xin_max=xin_max,
        out_max=out_max,
        n_counters=n_ctr,
        kinds=ops[:, 12] & 7,
        peer=peer_limit is not None,
        host_io=host_io,
        arena_elems=arena_elems,
        stage_elems=stage_elems,
        mr_segs=np.asarray(mr_segs, dtype=np.int64).reshape(-1, MR_FIELDS),
        mr_ranges=np.asarray(mr_ranges, dtype=np.int32).reshape(-1, MR_RANGE_FIELDS),
        bulk_only=bulk_only,
    )
