"""Static bounds validation of every program the packer emits (compute-sanitizer stand-in,
oracle/program_check.py): golden operators in every program variant -- single GPU, host-I/O,
multi-RHS re-chunked, W-way partitions (launch A + B) and peer-exchange partitions -- and
BASELINE configs 1-2 at full size."""

import pytest

from conftest import GOLDEN_NAMES, load_golden


def _variants(packed):
    from paper_2405_15573_b200.packer import MR_ROWS

    extra = []
    fwd, adj = packed.io_programs()
    for adj_, p in ((False, fwd), (True, adj)):
        if p is not None:
            extra.append((adj_, p, packed.work_len))
    f, a, wl = packed.programs(rows_per_chunk=MR_ROWS, far_rows=MR_ROWS)
    extra += [(False, f, wl), (True, a, wl)]
    return extra


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_golden_programs_in_bounds(name):
    from program_check import check_packed

    from paper_2405_15573_b200.packer import pack

    u, _ = load_golden(name)
    p = pack(u)
    assert check_packed(p, _variants(p)) >= 4
    for world in (2, 3):
        for peer in (False, True):
            for r in range(world):
                check_packed(p.for_rank(r, world, peer=peer))


@pytest.mark.parametrize("cfg", [1, 2])
def test_config_programs_in_bounds(cfg):
    from program_check import check_packed

    from paper_2405_15573_b200 import workloads
    from paper_2405_15573_b200.packer import pack

    p = pack(workloads.build_operator(cfg))
    check_packed(p, _variants(p))
    for r in range(4):
        check_packed(p.for_rank(r, 4, peer=True))


def test_checker_catches_corruption():
    from program_check import ProgramError, check_packed

    from paper_2405_15573_b200.packer import pack

    u, _ = load_golden("helm400")
    p = pack(u)
    i = int(p.fwd.pieces.shape[0] // 2)
    p.fwd.pieces[i, 0] = len(p.arena)  # a bulk copy past the arena
    with pytest.raises(ProgramError):
        check_packed(p)


def test_h_programs_in_bounds():
    """H-format programs, including the windowed-input FAR ops (OP_XWIN) of config 2."""
    import glob
    import os

    from conftest import GOLDEN
    from program_check import check_packed

    from paper_2405_15573_b200 import workloads
    from paper_2405_15573_b200.packer import OP_XWIN
    from paper_2405_15573_b200.packer_h import pack_h
    from paper_2405_15573_b200.uh_io import load_h

    for path in sorted(glob.glob(os.path.join(GOLDEN, "h_*.npz"))):
        check_packed(pack_h(load_h(path)[0]))
    import dataclasses

    from paper_2405_15573_b200.packer_h import _window_inputs

    p = pack_h(workloads.build_h_operator(2))  # 1 GB: packed without windows; window it here
    w = dataclasses.replace(p, fwd=_window_inputs(dataclasses.replace(p.fwd, ops=p.fwd.ops.copy()), 704),
                            adj=_window_inputs(dataclasses.replace(p.adj, ops=p.adj.ops.copy()), 704))
    assert w.fwd.xwin and w.adj.xwin and w.fwd.xin_max <= 704
    assert ((w.fwd.ops[:, 12] & OP_XWIN) != 0).sum() > 0
    check_packed(w)
