"""Peer-exchange partition (pack(peer=True)) on the CPU.

One program per rank and direction; the producers of a rank's y_t / u_t store them into
every rank's work buffer (RUN_PEER) and signal every rank's counters (OP_PEER); Z ops wait on
remote counters with the owner's producer count.  ``oracle/packed_vm.vm_peer_matvec`` runs
all ranks in one process with monotonic counters (epoch e waits for e x count), executing
each rank's tickets in order while their waits are met: a missing wait reads zeros (first
epoch) and fails the 1e-12 check, a wrong count deadlocks (assertion)."""

import numpy as np
import pytest

from conftest import load_golden, rel

NAMES = ["ico2_helm_compress", "uh800_laplace", "rect_sphere", "two_cloud", "degenerate", "no_admissible", "helm400"]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name", NAMES)
def test_peer_programs_match_reference(name, world):
    from packed_vm import vm_peer_matvec
    from paper_2405_15573_b200.packer import pack

    u, ex = load_golden(name)
    packs = [pack(u, rank=r, world=world, peer=True) for r in range(world)]
    for adjoint, vk, rk in ((False, "vf_0", "ref_fwd_0"), (True, "va_0", "ref_adj_0")):
        w = vm_peer_matvec(packs, ex[vk], adjoint=adjoint, epochs=2)
        assert rel(w, ex[rk]) <= 1e-12, (name, world, adjoint)


def test_peer_program_structure():
    """Shares add up to the whole operator; exchange outputs are plain stores of P1/RED/U ops
    inside the exchange region; every remote wait names a counter another rank signals."""
    from paper_2405_15573_b200.packer import (
        KIND_P1, KIND_RED, KIND_U, OP_PEER, RUN_PEER, pack,
    )

    u, _ = load_golden("ico2_helm_compress")
    world = 3
    total = pack(u).bytes_alg // 16
    for adjoint in (False, True):
        packs = [pack(u, rank=r, world=world, peer=True) for r in range(world)]
        progs = [p.adj if adjoint else p.fwd for p in packs]
        assert all(pr.peer and pr.part_b is None for pr in progs)
        share = sum(pr.arena_elems for pr in progs)
        assert total <= share <= 1.1 * total
        signalled = [set() for _ in range(world)]
        for r, pr in enumerate(progs):
            off, ex_len = packs[r].exchange["adj" if adjoint else "fwd"]
            for i in range(pr.n_ops):
                peer_runs = [q for q in pr.runs[pr.ops[i, 6] : pr.ops[i, 7]] if q[4] & RUN_PEER]
                assert bool(peer_runs) == bool(pr.ops[i, 12] & OP_PEER)
                if peer_runs:
                    assert pr.kinds[i] in (KIND_P1, KIND_RED, KIND_U)
                    for buf, o, ln, _dst, fl in peer_runs:
                        # this rank's block of the exchange region, plain stores
                        assert r * ex_len <= o - off and o - off + ln <= (r + 1) * ex_len and fl == RUN_PEER
                    signalled[r].update(int(c) for c in pr.sigs[pr.ops[i, 10] : pr.ops[i, 11]])
        for r, pr in enumerate(progs):
            local = {int(c) for i in range(pr.n_ops) for c in pr.sigs[pr.ops[i, 10] : pr.ops[i, 11]]}
            remote = set().union(*[signalled[q] for q in range(world) if q != r])
            for c, _n in pr.waits:
                assert int(c) in local or int(c) in remote


def test_peer_single_rank_is_plain_program():
    from paper_2405_15573_b200.packer import pack

    u, _ = load_golden("helm400")
    p = pack(u, peer=True)
    assert not p.fwd.peer and not (p.fwd.ops[:, 12] & 16).any()
    np.testing.assert_array_equal(p.fwd.ops, pack(u).fwd.ops)


def test_for_rank_equals_pack():
    from paper_2405_15573_b200.packer import pack

    u, _ = load_golden("ico2_helm_compress")
    base = pack(u, rank=0, world=3, peer=True)
    for r in (1, 2):
        a, b = base.for_rank(r, 3, peer=True), pack(u, rank=r, world=3, peer=True)
        assert a.work_len == b.work_len and a.exchange == b.exchange
        for name in ("ops", "pieces", "runs", "waits", "sigs", "fused_order"):
            np.testing.assert_array_equal(getattr(a.fwd, name), getattr(b.fwd, name))
            np.testing.assert_array_equal(getattr(a.adj, name), getattr(b.adj, name))
    assert base.for_rank(0, 1).fwd.n_ops == pack(u).fwd.n_ops
