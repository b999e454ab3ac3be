"""Versioned on-disk format of a PACKED operator.

``uh_io`` stores the reference-level objects (trees, bases, coefficients); this stores what
the device engines consume -- the HBM arena and the op programs (index tables, dependency
counters, multi-RHS segments) -- so a config is packed once and later loaded straight into
``DeviceOperator`` (no tree walk, no re-pack).  One ``.npz``:

  meta        JSON: format version, shapes, dtype, byte accounting, partition, exchange
  arena       complex128 (the packed operator, packer.py layout)
  {prog}_*    every Program array (ops, segs, pieces, runs, waits, sigs, fused_order, kinds,
              mr_segs, mr_ranges, phases) plus its scalars in meta; prog = fwd / adj, their
              multi-GPU launch-B halves fwd_b / adj_b, and every re-chunked multi-RHS program
              pair mr{rows}x{far}_fwd / _adj
"""

from __future__ import annotations

import json

import numpy as np

from .packer import PackedOperator, Program

__all__ = ["save_packed", "load_packed", "FORMAT_VERSION"]

FORMAT_VERSION = 1
_ARRAYS = ("ops", "segs", "pieces", "runs", "waits", "sigs", "fused_order", "kinds", "mr_segs", "mr_ranges", "mr_lds")
_SCALARS = ("in_max", "xin_max", "out_max", "n_counters", "zero_output", "arena_elems", "stage_elems", "w_order")


def _put(out, meta, name, prog: Program):
    for a in _ARRAYS:
        out[f"{name}_{a}"] = np.asarray(getattr(prog, a))
    out[f"{name}_phases"] = np.asarray(prog.phases, dtype=np.int64).reshape(-1, 2)
    meta["programs"][name] = {k: (bool(v) if isinstance(v, (bool, np.bool_)) else int(v))
                              for k, v in ((k, getattr(prog, k)) for k in _SCALARS)}
    if prog.part_b is not None:
        meta["programs"][name]["part_b"] = name + "_b"
        _put(out, meta, name + "_b", prog.part_b)


def _get(z, meta, name) -> Program:
    sc = meta["programs"][name]
    prog = Program(
        ops=z[f"{name}_ops"],
        segs=z[f"{name}_segs"],
        pieces=z[f"{name}_pieces"],
        runs=z[f"{name}_runs"],
        waits=z[f"{name}_waits"],
        sigs=z[f"{name}_sigs"],
        phases=[tuple(int(v) for v in r) for r in z[f"{name}_phases"]],
        fused_order=z[f"{name}_fused_order"],
        in_max=sc["in_max"],
        xin_max=sc["xin_max"],
        out_max=sc["out_max"],
        n_counters=sc["n_counters"],
        kinds=z[f"{name}_kinds"],
        zero_output=bool(sc["zero_output"]),
        w_order=bool(sc.get("w_order", False)),
        arena_elems=sc["arena_elems"],
        stage_elems=sc["stage_elems"],
        mr_segs=z[f"{name}_mr_segs"],
        mr_ranges=z[f"{name}_mr_ranges"],
        mr_lds=z[f"{name}_mr_lds"],
    )
    if "part_b" in sc:
        prog.part_b = _get(z, meta, sc["part_b"])
    return prog


def save_packed(path: str, p: PackedOperator, *, mr_chunks=None) -> None:
    """Write ``p``; ``mr_chunks`` (list of (rows, far_rows)) re-chunked programs are built
    first when the pack still has its index structure (default: the multi-RHS chunking)."""
    from .packer import MR_ROWS

    if mr_chunks is None:
        mr_chunks = [(MR_ROWS, MR_ROWS)] if (p.geo is not None and p.world == 1) else []
    for rows, far in mr_chunks:
        p.programs(rows_per_chunk=rows, far_rows=far)
    meta = {
        "format": "uhmv-packed",
        "version": FORMAT_VERSION,
        "n_rows": p.n_rows,
        "n_cols": p.n_cols,
        "dtype": np.dtype(p.dtype).str,
        "work_len": p.work_len,
        "n_adm": p.n_adm,
        "n_dense": p.n_dense,
        "bytes_alg": p.bytes_alg,
        "bytes_arena": p.bytes_arena,
        "storage": p.storage,
        "rank": p.rank,
        "world": p.world,
        "part": None if p.part is None else {k: (np.asarray(v).tolist() if not np.isscalar(v) else int(v)) for k, v in p.part.items()},
        "exchange": {k: [int(a) for a in v] for k, v in p.exchange.items()},
        "programs": {},
        "rechunked": [],
    }
    out = {"arena": p.arena}
    _put(out, meta, "fwd", p.fwd)
    _put(out, meta, "adj", p.adj)
    for (rows, far), (f, a, wl) in sorted(p.rechunked.items()):
        tag = f"mr{rows}x{far}"
        _put(out, meta, tag + "_fwd", f)
        _put(out, meta, tag + "_adj", a)
        meta["rechunked"].append([rows, far, int(wl), tag])
    out["meta"] = np.array(json.dumps(meta))
    np.savez(path, **out)


def load_packed(path: str) -> PackedOperator:
    with np.load(path, allow_pickle=False) as z:
        meta = json.loads(str(z["meta"]))
        if meta.get("format") != "uhmv-packed" or meta.get("version") != FORMAT_VERSION:
            raise ValueError(f"{path}: not a uhmv packed operator of format version {FORMAT_VERSION}")
        z = {k: z[k] for k in z.files}
    part = meta["part"]
    if part is not None:
        part = {k: (np.asarray(v, dtype=np.int64) if isinstance(v, list) else v) for k, v in part.items()}
    p = PackedOperator(
        n_rows=meta["n_rows"],
        n_cols=meta["n_cols"],
        dtype=np.dtype(meta["dtype"]),
        arena=z["arena"],
        work_len=meta["work_len"],
        fwd=_get(z, meta, "fwd"),
        adj=_get(z, meta, "adj"),
        n_adm=meta["n_adm"],
        n_dense=meta["n_dense"],
        bytes_alg=meta["bytes_alg"],
        bytes_arena=meta["bytes_arena"],
        storage=meta["storage"],
        rank=meta["rank"],
        world=meta["world"],
        part=part,
        exchange={k: tuple(v) for k, v in meta["exchange"].items()},
    )
    for rows, far, wl, tag in meta["rechunked"]:
        p.rechunked[(rows, far)] = (_get(z, meta, tag + "_fwd"), _get(z, meta, tag + "_adj"), wl)
    return p
