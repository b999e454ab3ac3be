"""Packed layout + op programs (P0 packer) checked on the CPU with the NumPy VM.

The VM (oracle/packed_vm.py) walks the arena and op tables exactly as the CUDA kernel
does; matching the reference's stored outputs here pins the layout before any GPU
run.  Structure gate G6: packed block ranges and slabs equal the
reference objects bit for bit.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel, views
from packed_vm import vm_matvec
from paper_2405_15573_b200.packer import (
    BUF_ARENA,
    BUF_WORK,
    HCOLS_MAX,
    KIND_FAR,
    KIND_NEAR,
    MODE_N,
    MODE_S,
    RUN_ATOMIC,
    pack,
)

TOL = 1e-12


@pytest.mark.parametrize("order,engine", [("phased", "segs"), ("fused", "segs"), ("fused", "pieces")])
def test_vm_matches_reference(golden, order, engine):
    name, u, ex = golden
    for vname, view, pfx in views():
        p = pack(view(u))
        for k in range(int(ex["nvec"])):
            w = vm_matvec(p, ex[f"vf_{k}"], order=order, engine=engine)
            assert rel(w, ex[f"{pfx}_fwd_{k}"]) <= TOL, (name, vname, order)
            w = vm_matvec(p, ex[f"va_{k}"], adjoint=True, order=order, engine=engine)
            assert rel(w, ex[f"{pfx}_adj_{k}"]) <= TOL, (name, vname, order, "adj")


def test_pieces_tile_stages(golden):
    """Bulk-kernel pieces: stages never overflow, begin/end flags pair up, every arena
    element of every segment is covered exactly once."""
    from paper_2405_15573_b200.packer import BULK_HCOLS_MAX, PI_BEGIN, PI_DIRECT, PI_END, PI_XSTAGE, STAGE_ELEMS

    name, u, ex = golden
    p = pack(u)
    for prog in (p.fwd, p.adj):
        for i in range(prog.n_ops):
            pcs = prog.pieces[prog.ops[i, 13] : prog.ops[i, 14]]
            open_ = False
            fill = 0
            for m_off, ld, rows, cols, mode, in_off, out_off, info in pcs:
                if mode in (1, 2):
                    assert cols <= BULK_HCOLS_MAX  # register slots of an H/S group
                if info & PI_DIRECT:
                    continue
                xw = (cols if mode in (0, 3) else rows) if info & PI_XSTAGE else 0
                if info & PI_BEGIN:
                    assert not open_
                    open_ = True
                    stage = (int(info) >> 32) & 0xFFFFFF
                    assert 0 < stage <= prog.stage_elems
                    fill = 0
                assert open_
                assert (int(info) & 0xFFFFFF) == fill
                fill += rows * cols + xw
                assert fill <= prog.stage_elems
                if info & PI_END:
                    assert fill == stage
                    open_ = False
            assert not open_


def test_program_invariants(golden):
    name, u, ex = golden
    p = pack(u)
    for prog, n_out in ((p.fwd, p.n_rows), (p.adj, p.n_cols)):
        # fused order is a permutation; every wait targets an earlier ticket
        assert sorted(prog.fused_order.tolist()) == list(range(prog.n_ops))
        pos = np.empty(prog.n_ops, dtype=np.int64)
        pos[prog.fused_order] = np.arange(prog.n_ops)
        producers = {}
        for i in range(prog.n_ops):
            sb, se = prog.ops[i, 10], prog.ops[i, 11]
            for c in prog.sigs[sb:se]:
                producers.setdefault(int(c), []).append(i)
        for i in range(prog.n_ops):
            wb, we = prog.ops[i, 8], prog.ops[i, 9]
            for c, cnt in prog.waits[wb:we]:
                ps = producers.get(int(c), [])
                assert len(ps) == cnt, (name, i, c)
                assert all(pos[q] < pos[i] for q in ps)
        # w is zeroed by the launcher; each entry gets at most one NEAR and one FAR atomic add
        # (two addends onto zero: order-independent), and nothing else writes w
        # -- or, ordered output (prog.w_order, no memset): every entry is STORED once (by its NEAR
        # op, or by its FAR op on a leaf without nearfield) and a FAR op that adds (plain
        # read-modify-write) waits for every NEAR op storing its rows, all on earlier tickets
        per_kind = {KIND_NEAR: np.zeros(n_out, dtype=np.int64), KIND_FAR: np.zeros(n_out, dtype=np.int64)}
        stores = np.zeros(n_out, dtype=np.int64)
        storer = {}
        assert prog.zero_output == (not prog.w_order)
        for i in range(prog.n_ops):
            ob, oe = prog.ops[i, 6], prog.ops[i, 7]
            for buf, off, ln, dst, flags in prog.runs[ob:oe]:
                if buf == 3:
                    assert prog.kinds[i] in per_kind
                    per_kind[int(prog.kinds[i])][off : off + ln] += 1
                    if not prog.w_order:
                        assert flags == RUN_ATOMIC
                    elif flags == 0:
                        stores[off : off + ln] += 1
                        for r in range(off, off + ln):
                            storer[r] = i
                    else:
                        assert flags == 1 and prog.kinds[i] == KIND_FAR
        assert (per_kind[KIND_NEAR] <= 1).all() and (per_kind[KIND_FAR] <= 1).all()
        if prog.w_order:
            assert (stores == 1).all()
            for i in range(prog.n_ops):
                ob, oe = prog.ops[i, 6], prog.ops[i, 7]
                for buf, off, ln, dst, flags in prog.runs[ob:oe]:
                    if buf == 3 and flags == 1:
                        waited = {q for c, _ in prog.waits[prog.ops[i, 8]:prog.ops[i, 9]] for q in producers.get(int(c), [])}
                        assert {storer[r] for r in range(off, off + ln)} <= waited
        # segment limits the kernel relies on
        segs = prog.segs
        hmask = segs[:, 5] != MODE_N
        assert (segs[hmask, 3] <= HCOLS_MAX).all()
        assert ((segs[:, 1] == BUF_WORK) == (segs[:, 5] == MODE_S)).all()
        assert (segs[:, 1] == BUF_ARENA).sum() + (segs[:, 1] == BUF_WORK).sum() == len(segs)
        assert (segs[:, 2] > 0).all() and (segs[:, 3] > 0).all()
        # slabs stay inside the arena
        arena_seg = segs[segs[:, 1] == BUF_ARENA]
        last = arena_seg[:, 0] + (arena_seg[:, 2] - 1) * arena_seg[:, 4] + arena_seg[:, 3]
        assert (last <= p.arena.size).all()


def test_structure_bit_exact(golden):
    """G6: every packed slab is the reference array bit for bit; ranges match block_ranges."""
    name, u, ex = golden
    p = pack(u)
    bct = u.bct
    # dense slabs: find each dense block through the forward NEAR ops
    prog = p.fwd
    seen = 0
    for i in np.nonzero(prog.kinds == KIND_NEAR)[0]:
        sb, se = prog.ops[i, 4], prog.ops[i, 5]
        ib = prog.ops[i, 2]
        for s in prog.segs[sb:se]:
            m_off, _, rows, cols, ld = s[:5]
            slab = p.arena[m_off + np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]]
            # locate the block by its column range
            run = [r for r in prog.runs[ib : prog.ops[i, 3]] if r[3] == s[6]][0]
            c_lo, c_len = run[1], run[2]
            out = [r for r in prog.runs[prog.ops[i, 6] : prog.ops[i, 7]]][0]
            r_lo = out[1]
            matches = [
                b for b in u.dense
                if bct.block_ranges(b)[2] == c_lo and bct.block_ranges(b)[3] == c_lo + c_len
                and bct.block_ranges(b)[0] <= r_lo < bct.block_ranges(b)[1]
            ]
            assert len(matches) == 1
            b = matches[0]
            r0 = r_lo - bct.block_ranges(b)[0]
            ref = np.asarray(u.dense[b], dtype=np.complex128)[r0 : r0 + rows]
            assert np.array_equal(slab, ref)
            seen += rows * cols
    assert seen == sum(d.size for d in u.dense.values())
    # cluster bases: reassembled from the leaf stacks, bit for bit
    from paper_2405_15573_b200.packer import unstack_basis

    for which, cmap, basis in (("U", bct.row_map, u.row_basis), ("V", bct.col_map, u.col_basis)):
        for c in cmap:
            m = np.asarray(basis.matrices[c], dtype=np.complex128)
            if m.shape[1] == 0:
                continue
            assert np.array_equal(unstack_basis(p.arena, p.geo, which, c), m), (which, c)
    # and every FAR op reads one contiguous stacked slab: the rows of all ancestor bases
    for i in np.nonzero(prog.kinds == KIND_FAR)[0]:
        segs = prog.segs[prog.ops[i, 4] : prog.ops[i, 5]]
        assert len({int(q[4]) for q in segs}) == 1  # one leaf stack (panel splits share its ld)


def test_bytes_accounting(golden):
    name, u, ex = golden
    p = pack(u)
    bases = sum(
        u.row_basis.matrices[s].size for s in u.bct.row_map
    ) + sum(u.col_basis.matrices[t].size for t in u.bct.col_map)
    coup = 0
    for b, pair in u.coeffs.items():
        blk = u.bct.nodes[b]
        ls = u.row_basis.matrices[blk.row].shape[1]
        lt = u.col_basis.matrices[blk.col].shape[1]
        k = pair.s_x.shape[1]
        coup += min(k * (ls + lt), ls * lt)
    dense = sum(d.size for d in u.dense.values())
    assert p.bytes_alg == 16 * (bases + coup + dense)
    # the arena is the algorithmic bytes plus 128-B alignment padding only
    # (+ what small operators store beyond the minimum: product-biased forms, the adjoint copy)
    extra = p.storage["form_extra"] + p.storage["adjoint_copy"]
    assert p.bytes_arena >= p.bytes_alg + extra
    assert p.bytes_arena - p.bytes_alg - extra <= 128 * (len(u.coeffs) + len(u.dense) + 5 * len(u.bct.nodes) + 8)
    os.environ["UHMV_ADJ_COPY"] = "0"
    try:
        q = pack(u, factor_bias=1.0)  # the byte minimum: nothing extra
    finally:
        del os.environ["UHMV_ADJ_COPY"]
    assert q.storage["form_extra"] == 0 and q.storage["adjoint_copy"] == 0
    assert pack(u, factor_bias=1.0).storage["form_extra"] == 0  # (default from 1 GB on: the copy only)
    assert q.bytes_arena - q.bytes_alg <= 128 * (len(u.coeffs) + len(u.dense) + 4 * len(u.bct.nodes) + 8)


def test_vm_matmat_multi_rhs(golden):
    """Multi-RHS segments (one input source each) == the reference's column loop."""
    from matvec_oracle import oracle_matvec_uh
    from packed_vm import vm_matmat

    name, u, ex = golden
    p = pack(u)
    rng = np.random.default_rng(11)
    for adjoint in (False, True):
        n_in = u.shape[0] if adjoint else u.shape[1]
        V = rng.standard_normal((n_in, 5)) + 1j * rng.standard_normal((n_in, 5))
        W = vm_matmat(p, V, adjoint=adjoint)
        ref = np.stack([oracle_matvec_uh(u, V[:, j], adjoint=adjoint) for j in range(5)], axis=1)
        assert rel(W, ref) <= TOL, (name, adjoint)


@pytest.mark.parametrize("name", ["helm400", "degenerate", "rect_sphere", "two_cloud", "h_ico2_helm"])
def test_mr_segments_fit_tma_rows(name):
    """Multi-RHS arena segments never wrap a TMA row: with (row, col) = divmod(m_off, ld),
    col + cols <= ld (matrices start at multiples of their ld), and every segment's map index
    points at its own ld."""
    from paper_2405_15573_b200.packer import MODE_S, MR_ROWS, MR_TMAP_SHIFT

    if name.startswith("h_"):
        from paper_2405_15573_b200.packer_h import pack_h
        from paper_2405_15573_b200.uh_io import load_h

        h, _ = load_h(os.path.join(GOLDEN, f"{name}.npz"))
        progs = [pack_h(h).fwd, pack_h(h).adj]
    else:
        u, _ = load_golden(name)
        p = pack(u)
        progs = [p.fwd, p.adj] + list(p.programs(rows_per_chunk=MR_ROWS, far_rows=MR_ROWS)[:2])
    for prog in progs:
        for m_off, ld, rows, cols, mode, _b, _a, _o in prog.mr_segs.tolist():
            if mode & 0xFF == MODE_S:
                continue
            assert m_off % ld + cols <= ld, (m_off, ld, cols)
            assert prog.mr_lds[mode >> MR_TMAP_SHIFT] == ld


@pytest.mark.parametrize("name", ["helm400", "ico2_helm_compress", "rect_sphere"])
def test_small_stages_split_wide_rows(name):
    """With tiny stages every wide N row is cut into column panels and every wide H piece into
    column groups; the pieces program still computes the reference's outputs."""
    u, ex = load_golden(name)
    p = pack(u, stage_elems=96)
    for prog in (p.fwd, p.adj):
        pcs = prog.pieces
        assert (pcs[:, 3][np.isin(pcs[:, 4], (0, 3))] <= 48).all()
    for adjoint, vk, rk in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
        w = vm_matvec(p, ex[vk], adjoint=adjoint, order="fused", engine="pieces")
        assert rel(w, ex[rk]) <= TOL


def test_host_io_programs():
    """Host-I/O variant (uhmv_matvec_host with pinned buffers): same results as the plain
    program in the VM; P1 ops publish x (OP_XHOST, one input run), NEAR ops wait for it
    (OP_XWAIT), and every output leaf is drained exactly once -- its drain descriptor (the run
    after the op's output cover) carries the leaf's NEAR + FAR op count."""
    from conftest import GOLDEN_NAMES, load_golden, rel
    from packed_vm import run_program
    from paper_2405_15573_b200.packer import (
        BUF_HOSTW, BUF_X, KIND_FAR, KIND_NEAR, KIND_P1, OP_DRAIN, OP_XHOST, OP_XWAIT, pack,
    )

    n_checked = 0
    for name in GOLDEN_NAMES:
        u, ex = load_golden(name)
        p = pack(u)
        for adjoint, prog, vk, rk in zip((False, True), p.io_programs(), ("vf_0", "va_0"), ("ref_fwd_0", "ref_adj_0")):
            if prog is None:
                continue
            n_checked += 1
            assert prog.host_io
            x = np.asarray(ex[vk], dtype=np.complex128)
            n_out = p.n_cols if adjoint else p.n_rows
            w = np.zeros(n_out, dtype=np.complex128)
            run_program(prog, p.arena, np.zeros(p.work_len, dtype=np.complex128), x, w, order="fused", engine="pieces")
            assert rel(w, ex[rk]) <= 1e-12
            drains = {}
            covered = np.zeros(p.n_rows if not adjoint else p.n_cols, dtype=int)
            for i in range(prog.n_ops):
                f, k = int(prog.ops[i, 12]), int(prog.kinds[i])
                if k == KIND_P1:
                    assert f & OP_XHOST
                    rr = prog.runs[prog.ops[i, 2] : prog.ops[i, 3]]
                    assert len(rr) == 1 and rr[0][0] == BUF_X
                if k == KIND_NEAR:
                    assert f & OP_XWAIT and f & OP_DRAIN
                if k in (KIND_NEAR, KIND_FAR):
                    assert f & OP_DRAIN
                    d = prog.runs[prog.ops[i, 7]]
                    assert d[0] == BUF_HOSTW
                    key = (int(d[1]), int(d[2]), int(d[3]))
                    drains.setdefault(key, [int(d[4]), 0])[1] += 1
            for (lo, ln, _c), (expect, seen) in drains.items():
                assert expect == seen
                covered[lo : lo + ln] += 1
            n_out_rows = p.n_cols if adjoint else p.n_rows
            assert (covered[:n_out_rows] == 1).all()
    assert n_checked >= 8
