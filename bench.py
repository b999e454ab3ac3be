"""Benchmark: uniform-H matvecs/s (and effective HBM GB/s, roofline fraction) on B200.

One "step" = one uniform-H matrix-vector product over the whole operator of the chosen
BASELINE config (default: config 3, N=81920 -- the config BASELINE.json quotes at
1/2/4/8 B200), x already resident in HBM.  See DESIGN.md §Measurement.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--mode fused|phased]
  python bench.py --impl reference ...   # the reference algorithm on the host CPU

Under torchrun (N>1) every rank owns a contiguous slice of output leaves (row-cluster
partition); the y/u coefficients are exchanged inside the one kernel per
rank over NVLink peer mappings (``--exchange auto``: when every rank can map its peers and
the first matvecs agree with the NCCL path; else one NCCL all-gather between two launches);
time = max over ranks; value = whole-job matvecs/s.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3, help="BASELINE config 1-5 (5 = config 3 x 64 RHS)")
    ap.add_argument("--nrhs", type=int, default=64, help="right-hand sides of config 5")
    ap.add_argument("--mode", default="bulk", choices=["bulk", "fused", "phased"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--adjoint", action="store_true")
    ap.add_argument("--view", default="full", choices=["full", "far", "near"], help="diagnostics: parity view")
    ap.add_argument("--format", default="uh", choices=["uh", "h", "sym"],
                    help="uh: uniform H-matrix (the hot path); h: the source H-matrix (matvec_h)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "peer"],
                    help="multi-GPU y/u exchange: NCCL all-gather between two launches, or peer stores "
                         "over NVLink inside one launch per rank")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="diagnostics (1 GPU): run a W-rank peer-exchange partition in one launch, "
                         "each rank on 1/W of the SMs")
    ap.add_argument("--l2", default="auto", choices=["auto", "hot"],
                    help="auto: flush L2 between steps when the operator fits in ~4x L2; hot: never "
                         "(the L2-resident number SURVEY §8d asks for at config 1)")
    ap.add_argument("--slice", default="",
                    help="predict multi-GPU scaling on ONE GPU: comma-separated world sizes W; each rank's NCCL-path "
                         "programs (launch A + launch B of the W-way row partition) run alone on the whole GPU")
    ap.add_argument("--slice-exchange", default="both", choices=["nccl", "peer", "both"],
                    help="--slice: the NCCL path (launch A + B) and/or the fused peer-exchange launch (remote "
                         "y/u counters pre-satisfied: the data of the other ranks assumed there when needed)")
    ap.add_argument("--ag-lat-us", type=float, default=15.0, help="--slice model: NCCL all-gather latency (us)")
    ap.add_argument("--ag-gbs", type=float, default=300.0, help="--slice model: NCCL all-gather bandwidth (GB/s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0)
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = (
        "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
        "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {
            "sm_mhz": float(np.median(sm)) if sm else None,
            "sm_max_mhz": float(max(smax)) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(u, x, sample_s: float):
    """The reference's own matvec_uh (or, without oracle/_ref, the oracle port) on the host
    cores, bounded to ~sample_s seconds: grid over (BLAS threads, workers) in {(1, 1), (all, 1),
    (1, all)}, best cell reported, every cell listed."""
    fn, kind, desc = reference_impl()
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    ncpu = os.cpu_count() or 1
    cells = []
    for threads, workers in sorted({(1, 1), (ncpu, 1), (1, ncpu)}):
        ctx = threadpool_limits(limits=threads) if threadpool_limits else None
        try:
            fn(u, x, workers=workers)  # warm-up, excluded
            ts = []
            t_end = time.perf_counter() + sample_s / 3
            while len(ts) < 3 or (time.perf_counter() < t_end and len(ts) < 50):
                t0 = time.perf_counter()
                fn(u, x, workers=workers)
                ts.append(time.perf_counter() - t0)
        finally:
            if ctx is not None:
                ctx.__exit__(None, None, None)
        cells.append({"blas_threads": threads, "workers": workers, "reps": len(ts),
                      "min_ms": min(ts) * 1e3, "median_ms": float(np.median(ts)) * 1e3})
    best = min(cells, key=lambda c: c["median_ms"])
    return {
        "value": 1e3 / best["median_ms"],
        "unit": "matvec/s",
        "cores": max(best["blas_threads"], best["workers"]),
        "cpu_model": cpu_model(),
        "host_cpus": ncpu,
        "kind": kind,
        "grid": cells,
        "sample": f"{best['reps']} full matvecs (median) after 1 warm-up per cell, {desc}; best of the "
        f"(BLAS threads, workers) grid",
    }


# SURVEY §8d algorithmic bytes per matvec (operator in its cheapest stored form + x + w), used
# only for the L2 policy so that both arms state the same config without touching the GPU
ALG_BYTES = {1: 99.2e6, 2: 445.0e6, 3: 2643.6e6, 4: 8031e6}
L2_BYTES = 126.5e6


def l2_policy(cfg: int, world: int, l2: str) -> tuple[bool, str]:
    """(flush?, config string): flush L2 between steps when one GPU's share of the operator
    is under 4x the L2, unless --l2 hot."""
    share = ALG_BYTES.get(cfg, ALG_BYTES[3]) / max(world, 1)
    if l2 == "hot":
        return False, "L2-hot: no flush between steps"
    if share < 4 * L2_BYTES:
        return True, "L2 flushed between steps (write + read of a 2x L2 buffer, untimed)"
    return False, f"no flush: {share / 1e9:.2f} GB of operator per GPU >> L2"


def make_config(args, world):
    from paper_2405_15573_b200 import workloads

    if args.config == 5:
        return {"workload": "cfg5_cfg3_operator_x_%d_rhs" % args.nrhs, "N": 81920, "nrhs": args.nrhs,
                "values": "seeded synthetic on the reference-built cfg3 structure and ranks",
                "parallelism": (f"{world} GPUs, each its own block of {args.nrhs} right-hand sides (no exchange)"
                                if world > 1 else "single GPU")}
    meta = workloads.CONFIGS[args.config]
    config = {
        "workload": meta["name"],
        "N": meta["N"],
        "values": "seeded synthetic on the reference-built structure"
        + (" and ranks (rank-profile surrogate)" if meta["kind"] == "profile" else " (BASELINE config 4 spec)"),
        "vector": "default_rng(0) complex Gaussian, tree order",
        "mode": args.mode,
        "adjoint": bool(args.adjoint),
        "parallelism": f"row-partition x{world}" if world > 1 else "single GPU",
        "l2": l2_policy(args.config, world, args.l2)[1],
    }
    if args.format == "h":
        config["format"] = "H-matrix (matvec_h, hmatrix.py:143-184), ranks of the reference's assemble_h"
    if args.format == "sym":
        config["format"] = ("symmetric single-triangle variant (paper Remark 4.5; a LABELLED variant, not the "
                            "reference's two-triangle operator): one basis, lower blocks only, every slab read once")
    if args.view != "full":
        config["view"] = args.view
    if args.emulate_ranks > 1:
        config["parallelism"] = (f"peer-exchange partition of {args.emulate_ranks} ranks emulated in one launch "
                                 f"on one GPU (1/{args.emulate_ranks} of the SMs each)")
    return config


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2405_15573_b200 import workloads

    config = make_config(args, world)
    if args.slice:
        run_slice(args, config)
        return
    if args.impl == "reference":
        run_reference(args, rank, world, config)
        return
    if args.config == 5:
        run_multi_rhs(args, world, rank, local_rank, config)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)

    t_build = time.perf_counter()
    if args.format == "sym":
        if args.adjoint or world > 1 or args.emulate_ranks > 1 or args.view != "full":
            raise SystemExit("--format sym: forward, single GPU, full view only")
        u = workloads.build_symmetric_operator(args.config)
    elif args.format == "uh":
        u = workloads.build_operator(args.config)
    else:
        u = workloads.build_h_operator(args.config)
    if args.view != "full":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from matvec_oracle import farfield_only, nearfield_only

        u = farfield_only(u) if args.view == "far" else nearfield_only(u)
    x_np = workloads.seeded_vector(u.shape[1], 0)
    from paper_2405_15573_b200.packer import pack

    if world > 1:
        from paper_2405_15573_b200.dist import make_distributed

        op, why = make_distributed(u, rank, world, device=dev, exchange=args.exchange)
        config["exchange"] = op.exchange
        config["exchange_choice"] = why
        packed = op.packed_local
    elif args.emulate_ranks > 1:
        from paper_2405_15573_b200.dist import PeerEmulation

        op = PeerEmulation(u, args.emulate_ranks, device=dev)
        packed = op.packs[0]
    else:
        from paper_2405_15573_b200.device import DeviceOperator

        if args.format == "h":
            from paper_2405_15573_b200.packer_h import pack_h

            packed = pack_h(u)
        elif args.format == "sym":
            from paper_2405_15573_b200.packer_sym import pack_sym

            packed = pack_sym(u)
        else:
            packed = pack(u)
        op = DeviceOperator(packed, device=dev)
    t_build = time.perf_counter() - t_build

    n_in = u.shape[0] if args.adjoint else u.shape[1]
    n_out = u.shape[1] if args.adjoint else u.shape[0]
    x = torch.from_numpy(x_np if not args.adjoint else workloads.seeded_vector(n_in, 0)).to(dev)
    stream = torch.cuda.current_stream(dev)

    def step(out=None):
        return op.matvec(x, adjoint=args.adjoint, mode=args.mode, out=out)

    out = step()
    flush, _ = l2_policy(args.config, world, args.l2)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(int(2 * l2_bytes) // 4 + 1024, dtype=torch.float32, device=dev) if flush else None
    flush_rd = torch.zeros(int(2 * l2_bytes) // 4 + 1024, dtype=torch.float32, device=dev) if flush else None

    def flush_l2():
        # write a buffer > L2, then read another one: the read evicts the dirty lines (their
        # write-back happens here, untimed) and leaves L2 cold and clean for the timed step
        flush_buf.zero_()
        flush_rd.sum()

    warmup = max(args.warmup, 3)
    for _ in range(warmup):
        if flush:
            flush_l2()
        step(out)
    torch.cuda.synchronize(dev)

    def timed(k):
        """k steps, CUDA events around every step's kernel(s) on the launching stream."""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        for i in range(k):
            if flush:
                flush_l2()
            starts[i].record(stream)
            step(out)
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        return np.array([s.elapsed_time(e) for s, e in zip(starts, ends)]) * 1e-3  # s

    # timed region: exactly K steps between barriers + synchronize, clocks sampled during it
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    per_step = timed(args.steps)
    if world > 1:
        torch.distributed.barrier()
    # the distribution SURVEY §8d asks for (median of >= 100 reps), when K is smaller
    dist_steps = per_step if args.steps >= 100 else np.concatenate([per_step, timed(100)])
    clk = clocks.stop()
    med_s, mean_s = float(np.median(per_step)), float(per_step.mean())
    med100 = float(np.median(dist_steps))
    if world > 1:
        t = torch.tensor([med_s, mean_s, med100], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        med_s, mean_s, med100 = (float(v) for v in t.tolist())

    # end to end through the reference-facing C-ABI call with host buffers (multi-GPU: the
    # same call gathers the output slices; time = max over ranks)
    xh = torch.from_numpy(x.cpu().numpy()).pin_memory()
    wh = torch.empty(n_out, dtype=torch.complex128).pin_memory()
    xh_np, wh_np = xh.numpy(), wh.numpy()
    for _ in range(10):  # includes the host-I/O vs copy-path choice (4 calls each)
        op.matvec_host(xh_np, adjoint=args.adjoint, out=wh_np, mode=args.mode)
    k_e2e = max(10, min(args.steps, 200))

    def wall(fn, k):
        if world > 1:
            torch.distributed.barrier()
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        te = float(np.median(ts))
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        return te

    te = wall(lambda: op.matvec_host(xh_np, adjoint=args.adjoint, out=wh_np, mode=args.mode), k_e2e)
    e2e = {
        "value": 1.0 / te,
        "unit": "matvec/s",
        "h2d_bytes_per_step": int(16 * n_in),
        "d2h_bytes_per_step": int(16 * n_out),
        "api": "uhmv_matvec_host (C ABI, pinned host x/w, H2D + kernels + D2H + sync; wall clock, median)",
    }
    choice = op.host_io_choice(args.adjoint) if hasattr(op, "host_io_choice") else None
    if choice is not None:
        e2e["path"] = ("host-I/O launch: x read over PCIe by the P1 ops, finished output leaves drained "
                       "to the pinned host buffer inside the kernel" if choice
                       else "H2D copy + launch + D2H copy (faster than the host-I/O launch here)")
    # the drop-in itself: matvec_uh(u, ndarray) as a reference caller makes it (pageable input,
    # a NEW output array every call, dtype promotion, validation), single GPU
    e2e_dropin = None
    if world == 1 and args.emulate_ranks <= 1 and args.view == "full":
        import paper_2405_15573_b200 as pk
        from paper_2405_15573_b200.matvec import register_device_operator

        register_device_operator(u, op)
        xr = (x_np if not args.adjoint else workloads.seeded_vector(n_in, 0)).copy()
        fn = {"h": pk.matvec_h, "sym": pk.matvec_uh_sym}.get(args.format, pk.matvec_uh)
        for _ in range(10):
            fn(u, xr, adjoint=args.adjoint)
        td = wall(lambda: fn(u, xr, adjoint=args.adjoint), k_e2e)
        e2e_dropin = {"value": 1.0 / td, "unit": "matvec/s", "h2d_bytes_per_step": int(16 * n_in),
                      "d2h_bytes_per_step": int(16 * n_out),
                      "api": f"paper_2405_15573_b200.{fn.__name__}(u, numpy array) -- the installed drop-in "
                             "(pageable input, new output array per call); wall clock, median"}

    peak, peak_kind = measured_peaks()
    alg_bytes_total = workloads.algorithmic_bytes(packed)
    value = 1.0 / med_s
    achieved = alg_bytes_total / world / med_s / 1e9  # per GPU
    traffic = (load_traffic(args.config) if args.format == "uh" and args.view == "full" and not args.adjoint
               else load_traffic(f"sym_cfg{args.config}" if args.format == "sym" else None))
    roofline = {
        "bound": "hbm",
        "achieved": achieved,
        "peak": peak,
        "unit": "GB/s",
        "frac": achieved / peak,
        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
        "frac_vs_8000_nominal": achieved / 8000.0,
        "traffic": traffic,
        "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                          "(profiles/ncu_traffic.json, same command)",
        "algorithmic_bytes_per_launch": int(alg_bytes_total / world),
        "reference_bytes_estimate": ref_bytes_estimate(args.config, u) if args.format != "sym" else None,
        "kernel": "bulk::uhmv_bulk_sym_kernel" if args.format == "sym" else
        "bulk::uhmv_bulk_peer_kernel" if (args.emulate_ranks > 1 or getattr(op, "exchange", "") == "peer") else
        {"bulk": "bulk::uhmv_bulk_kernel", "fused": "uhmv_fused_kernel"}.get(args.mode, "uhmv_phase_kernel (5 launches)"),
    }
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": "uniform-H matvecs/sec (effective HBM GB/s, roofline fraction)",
        "value": value,
        "unit": "matvec/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": warmup,
        "ms_per_step": med_s * 1e3,
        "ms_per_step_mean": mean_s * 1e3,
        "ms_per_step_median_100": med100 * 1e3,
        "reps_for_median_100": int(len(dist_steps)),
        "effective_gbs": achieved * world,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c128 (f64 complex)",
        "data": "synthetic",
        "config": config,
        "roofline": roofline,
        "exchange_bytes_per_rank": (16 * op.packed_local.exchange["adj" if args.adjoint else "fwd"][1]) if world > 1 else 0,
        "e2e": e2e,
        "e2e_dropin": e2e_dropin,
        "gpu_launches": args.steps * op.kernel_launches(args.adjoint, args.mode),
        "clocks": clk,
        "build_s": t_build,
        "launch": op.launch_info(args.adjoint, args.mode),
    }
    if os.environ.get("UHMV_PROFILE") and world == 1 and args.mode == "bulk":
        line["engine_cycles"] = op.profile(args.adjoint, args.mode)
    if world == 1 and not args.no_cpu_baseline and args.format == "uh":
        line["cpu_baseline"] = cpu_baseline(u, x_np, args.cpu_sample_s) if not args.adjoint else None
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_slice(args, config):
    """--slice W[,W...]: one-GPU predictor of the W-GPU row partition.

    For every rank r of a W-way partition (packer.partition_bounds, bytes-balanced) the rank's
    NCCL-path programs -- launch A (P1, RED, U, part of the nearfield), launch B (Z, the rest
    of the nearfield, FAR) -- run back to back ALONE on the whole B200, exactly the kernels that
    rank runs on its own GPU (the exchange region holds stale values: timing only).  Reports
    per-rank bytes and device time (median, L2 policy of a W-GPU run), the max/mean imbalance,
    and the predicted speed-up t1 / (max_r t_r + t_ag), t_ag = a modelled NCCL all-gather of
    the y/u exchange region (--ag-lat-us + bytes / --ag-gbs)."""
    import torch

    from paper_2405_15573_b200 import workloads
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    u = workloads.build_operator(args.config)
    packed = pack(u)
    base = DeviceOperator(packed, device=dev)
    n_in = u.shape[0] if args.adjoint else u.shape[1]
    x = torch.from_numpy(workloads.seeded_vector(n_in, 0)).to(dev)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(int(2 * l2_bytes) // 4 + 1024, dtype=torch.float32, device=dev)
    flush_rd = torch.zeros_like(flush_buf)
    steps = max(args.steps, 20)

    def timed(fn, flush):
        for _ in range(max(args.warmup, 3)):
            fn()
        ts = []
        for _ in range(steps):
            if flush:
                flush_buf.zero_()
                flush_rd.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize(dev)
        return float(np.median([a.elapsed_time(b) for a, b in ts])) * 1e-3

    out = torch.empty(u.shape[1] if args.adjoint else u.shape[0], dtype=torch.complex128, device=dev)
    t1 = timed(lambda: base.matvec(x, adjoint=args.adjoint, out=out), l2_policy(args.config, 1, args.l2)[0])
    b1 = workloads.algorithmic_bytes(packed)
    peak, _ = measured_peaks()
    res = {"metric": "one-GPU prediction of W-GPU uniform-H matvec scaling (rank programs run alone)",
           "config": config, "t1_ms": t1 * 1e3, "t1_frac": b1 / t1 / 1e9 / peak, "alg_bytes_1": b1,
           "ag_model": {"lat_us": args.ag_lat_us, "gbs": args.ag_gbs}, "worlds": []}
    for W in [int(v) for v in args.slice.split(",") if v.strip()]:
        flush = l2_policy(args.config, W, args.l2)[0]
        if args.slice_exchange in ("peer", "both"):
            res["worlds_peer"] = res.get("worlds_peer", []) + [_slice_peer(args, packed, base, x, W, flush, t1, peak)]
        if args.slice_exchange == "peer":
            continue
        ranks = []
        for r in range(W):
            pr = packed.for_rank(r, W)
            a = DeviceOperator(pr, device=dev, share_arena_with=base)
            b = DeviceOperator(pr, device=dev, programs=(pr.fwd.part_b, pr.adj.part_b), share_with=a)
            prog = pr.adj if args.adjoint else pr.fwd

            def step(a=a, b=b):
                a.matvec(x, adjoint=args.adjoint, out=out)
                b.matvec(x, adjoint=args.adjoint, out=out)

            t = timed(step, flush)
            nbytes = 16 * (prog.arena_elems + prog.part_b.arena_elems)
            ex_elems = pr.exchange["adj" if args.adjoint else "fwd"][1]
            ranks.append({"rank": r, "ms": t * 1e3, "bytes": nbytes, "frac": nbytes / t / 1e9 / peak,
                          "rows": [int(pr.part["row_bounds"][r]), int(pr.part["row_bounds"][r + 1])],
                          "exchange_bytes": 16 * int(ex_elems) * W})
            a.close()
            b.close()
            del a, b
        tmax = max(q["ms"] for q in ranks) * 1e-3
        bts = [q["bytes"] for q in ranks]
        ms = [q["ms"] for q in ranks]
        t_ag = args.ag_lat_us * 1e-6 + max(q["exchange_bytes"] for q in ranks) / (args.ag_gbs * 1e9)
        res["worlds"].append({
            "W": W, "ranks": ranks, "bytes_max_over_mean": max(bts) / (sum(bts) / W),
            "time_max_over_mean": max(ms) / (sum(ms) / W), "bytes_sum_over_1gpu": sum(bts) / packed.bytes_alg,
            "t_max_ms": tmax * 1e3, "t_allgather_model_ms": t_ag * 1e3,
            "predicted_speedup": t1 / (tmax + t_ag), "predicted_efficiency": t1 / (tmax + t_ag) / W,
            "predicted_speedup_no_exchange_cost": t1 / tmax,
        })
    print(json.dumps(res), flush=True)


def _slice_peer(args, packed, base, x, W, flush, t1, peak):
    """One rank of the fused peer-exchange path (``pack(peer=True)``: ONE launch per rank and
    matvec) run alone on the whole GPU: its own work / counters / done flags, the peers'
    buffers replaced by scratch, and before every epoch e the counters only OTHER ranks signal
    set to their final value (need x e) and the peers' done flags to e -- i.e. the remote y/u
    are taken to arrive by the time this rank needs them (the ranks run symmetric programs on
    equal shares, and the all-gather payload is ~1 MB against GBs of operator)."""
    import torch

    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.dist import _execute_peer, _peer_rank

    dev = base.device
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(int(2 * l2_bytes) // 4 + 1024, dtype=torch.float32, device=dev)
    flush_rd = torch.zeros_like(flush_buf)
    steps = max(args.steps, 20)
    ranks_out = []
    for r in range(W):
        pr = packed.for_rank(r, W, peer=True)
        op = DeviceOperator(pr, device=dev, share_arena_with=base)
        prog = pr.adj if args.adjoint else pr.fwd
        n_ctr = max(pr.fwd.n_counters, pr.adj.n_counters, 1)
        wl = max(pr.work_len, 1)
        own = (torch.zeros(2 * wl, dtype=torch.complex128, device=dev), torch.zeros(n_ctr, dtype=torch.int32, device=dev),
               torch.zeros(W, dtype=torch.int32, device=dev))
        dummy = (torch.zeros(2 * wl, dtype=torch.complex128, device=dev), torch.zeros(n_ctr, dtype=torch.int32, device=dev),
                 torch.zeros(W, dtype=torch.int32, device=dev))
        ranks = [_peer_rank(b[0].data_ptr(), wl, b[1].data_ptr(), b[2].data_ptr()) for b in
                 [own if q == r else dummy for q in range(W)]]
        signalled = set(int(c) for c in prog.sigs)
        need = {}
        for c, n in prog.waits:
            if int(c) not in signalled:
                need[int(c)] = max(need.get(int(c), 0), int(n))
        idx = torch.tensor(sorted(need), dtype=torch.long, device=dev)
        nv = torch.tensor([need[c] for c in sorted(need)], dtype=torch.int32, device=dev)
        n_out = packed.n_cols if args.adjoint else packed.n_rows
        out = torch.empty(n_out, dtype=torch.complex128, device=dev)
        stream = torch.cuda.current_stream(dev)
        epoch = 0
        ts = []
        for i in range(max(args.warmup, 3) + steps):
            epoch += 1
            if flush:
                flush_buf.zero_()
                flush_rd.sum()
            if len(need):
                own[1][idx] = nv * epoch
            own[2].fill_(epoch)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _execute_peer([op._plan], r, W, ranks, x, [out], args.adjoint, epoch, stream)
            b.record(stream)
            if i >= max(args.warmup, 3):
                ts.append((a, b))
        torch.cuda.synchronize(dev)
        t = float(np.median([a.elapsed_time(b) for a, b in ts])) * 1e-3
        nbytes = 16 * prog.arena_elems
        ranks_out.append({"rank": r, "ms": t * 1e3, "bytes": nbytes, "frac": nbytes / t / 1e9 / peak,
                          "remote_counters": len(need)})
        op.close()
        del op, own, dummy
    tmax = max(q["ms"] for q in ranks_out) * 1e-3
    bts = [q["bytes"] for q in ranks_out]
    return {"W": W, "exchange": "peer (one launch per rank, remote y/u pre-satisfied)", "ranks": ranks_out,
            "bytes_max_over_mean": max(bts) / (sum(bts) / W), "t_max_ms": tmax * 1e3,
            "predicted_speedup": t1 / tmax, "predicted_efficiency": t1 / tmax / W}


def ref_bytes_estimate(cfg, u=None):
    """The reference's own figure: storage_report_uh(u).bytes_estimate (uniform.py:559-584),
    computed by the reference itself (oracle/_ref) on the benchmarked operator, else the value
    stored in the config fixture by tools/make_workloads.py for the reference-built operator."""
    from paper_2405_15573_b200 import workloads

    if u is not None and hasattr(u, "coeffs") and os.path.isdir(os.path.join(REF_SITE, "uhm_kit")):
        if REF_SITE not in sys.path:
            sys.path.append(REF_SITE)
        from uhm_kit.uniform import storage_report_uh

        return int(storage_report_uh(u).bytes_estimate)
    try:
        with np.load(workloads.workload_path(cfg)) as z:
            return int(z["x_ref_bytes_estimate"]) if "x_ref_bytes_estimate" in z.files else None
    except (OSError, KeyError):
        return None


def dmma_peak(device_index: int):
    import ctypes

    from paper_2405_15573_b200 import _lib

    pk = ctypes.c_double()
    _lib.check(_lib.lib().uhmv_dmma_peak(device_index, ctypes.byref(pk)), "uhmv_dmma_peak")
    return pk.value


def run_multi_rhs(args, world, rank, local_rank, config):
    """BASELINE config 5: the config-3 operator applied to a block of nrhs seeded complex
    Gaussian right-hand sides on FP64 tensor cores (DMMA).  One step = one block product;
    value = right-hand sides per second (matvecs/s).  Roofline: FP64 tensor peak measured
    in-run (uhmv_dmma_peak)."""
    import torch

    from paper_2405_15573_b200 import workloads
    from paper_2405_15573_b200.device import DeviceOperator
    from paper_2405_15573_b200.packer import pack

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if world > 1:  # every rank applies the operator to its own block of right-hand sides
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    R = args.nrhs
    u = workloads.build_operator(3)
    packed = pack(u)
    op = DeviceOperator(packed, device=dev)
    n = u.shape[1]
    rng = np.random.default_rng(0 if world == 1 else [0, rank])
    Xh = rng.standard_normal((n, R)) + 1j * rng.standard_normal((n, R))
    X = torch.from_numpy(Xh).to(dev)
    op.matmat(X)
    for _ in range(max(args.warmup, 3)):
        op.matmat(X)
    torch.cuda.synchronize(dev)
    steps = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    for a, b in ev:
        a.record()
        op.matmat(X)
        b.record()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e-3
    if world > 1:  # time = max over ranks
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    flops = 8.0 * R * packed.bytes_alg / 16  # 4 real mul + 4 add per complex MAC
    peak = dmma_peak(dev.index)
    # e2e: pinned host block in, pinned host block out (H2D + kernel + D2H + sync, wall clock)
    Xp = torch.from_numpy(Xh).pin_memory()
    Wp = torch.empty((n, R), dtype=torch.complex128).pin_memory()
    Wd = torch.empty((n, R), dtype=torch.complex128, device=dev)

    Xp_np, Wp_np = Xp.numpy(), Wp.numpy()

    def e2e_step():  # C-ABI host call: column chunks pipelined (H2D || DMMA || D2H)
        op.matmat_host(Xp_np, out=Wp_np)

    for _ in range(2):
        e2e_step()
    te = time.perf_counter()
    ke = 10
    for _ in range(ke):
        e2e_step()
    te = (time.perf_counter() - te) / ke
    if world > 1:
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
        if rank != 0:
            dist.destroy_process_group()
            return
    line = {
        "metric": "uniform-H matvecs/sec (multi-RHS block, config 5)",
        "value": world * R / t,
        "unit": "matvec/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "weak" if world > 1 else "strong",
        "vs_baseline": None,
        "dtype": "c128 (f64 complex)",
        "data": "synthetic",
        "config": config,
        "roofline": {"bound": "tensor", "achieved": flops / t / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": flops / t / 1e12 / peak,
                     "peak_source": "uhmv_dmma_peak: measured DMMA m16n8k16 f64 throughput on this GPU "
                                    "(MEASURED_PEAKS.json has no FP64 entry)",
                     "traffic": load_traffic("cfg5") if R == 64 else None,
                     "tensor_pipe_active_pct": load_traffic("cfg5_dmma_pipe_active_pct") if R == 64 else None,
                     "tensor_pipe_source": "ncu smsp__pipe_tensor_subpipe_dmma_cycles_active (profiles/r02/ncu_full_mrtc_cfg5.json)",
                     "flops_per_launch": flops, "kernel": "mrtc::uhmv_mrtc_kernel"},
        "e2e": {"value": world * R / te, "unit": "matvec/s", "h2d_bytes_per_step": int(16 * n * R),
                "d2h_bytes_per_step": int(16 * n * R),
                "api": "uhmv_matmat_host (C ABI, pinned host X/W, 32-column chunks: H2D, DMMA product and "
                       "D2H of consecutive chunks overlap on three streams; wall clock)"},
        "gpu_launches": steps,
        "clocks": clk,
    }
    if os.environ.get("UHMV_PROFILE"):
        line["engine_cycles"] = op.profile_mr(R)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def load_traffic(cfg):
    """DRAM bytes per launch from the committed ncu --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = json.load(fh)
    v = d.get(cfg if isinstance(cfg, str) else f"cfg{cfg}") if cfg is not None else None
    return float(v) if v is not None else None


REF_SITE = os.path.join(ROOT, "oracle", "_ref", "site")


def reference_impl():
    """The CPU reference the GPU is compared with: the UNMODIFIED reference ``uhm_kit``
    (``uniform.matvec_uh``, uniform.py:476-556), installed into oracle/_ref by
    oracle/build_ref.sh and shipped with the repo; else the oracle port restating it."""
    if os.path.isdir(os.path.join(REF_SITE, "uhm_kit")):
        if REF_SITE not in sys.path:
            sys.path.append(REF_SITE)
        import uhm_kit.uniform

        fn = uhm_kit.uniform.matvec_uh
        if fn.__module__ != "uhm_kit.uniform":
            raise RuntimeError("uhm_kit.uniform.matvec_uh is patched (install() active): not the reference")
        return fn, "reference", "uhm_kit.uniform.matvec_uh (the unmodified reference, oracle/_ref/site)"
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from matvec_oracle import oracle_matvec_uh

    return oracle_matvec_uh, "port", "oracle/matvec_oracle.py (restates uniform.py:476-556)"


def run_reference(args, rank, world, config):
    """--impl reference: the reference's own matvec_uh on the host CPU, all host threads (BLAS
    threads = os.cpu_count(), workers=1: the reference's thread pool is GIL-bound);
    rank 0 only under torchrun.  Same warm-up count, config keys, metric and unit as the GPU
    arm; each step is one full matvec, the timed steps bounded to ~60 s of CPU work."""
    if rank != 0:
        return
    from paper_2405_15573_b200 import workloads

    fn, kind, desc = reference_impl()
    cfg = 3 if args.config == 5 else args.config  # config 5 = the config-3 operator, column loop
    u = workloads.build_operator(cfg)
    n_in = u.shape[0] if args.adjoint else u.shape[1]
    if args.config == 5:  # the reference has no block product: one matvec per right-hand side
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n_in, args.nrhs)) + 1j * rng.standard_normal((n_in, args.nrhs))
    else:
        X = workloads.seeded_vector(n_in, 0)[:, None]
    n_warm = max(args.warmup, 3)
    for i in range(n_warm):
        fn(u, X[:, i % X.shape[1]], adjoint=args.adjoint)
    ts = []
    t_all = time.perf_counter()
    for i in range(max(args.steps, 1)):
        t0 = time.perf_counter()
        fn(u, X[:, i % X.shape[1]], adjoint=args.adjoint)
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > 60.0:
            break
    med = float(np.median(ts))
    value = 1.0 / med
    ncpu = os.cpu_count() or 1
    line = {
        "impl": "reference",
        "metric": ("uniform-H matvecs/sec (multi-RHS block, config 5)" if args.config == 5
                   else "uniform-H matvecs/sec (effective HBM GB/s, roofline fraction)"),
        "value": value,
        "unit": "matvec/s",
        "n_gpus": world,
        "steps": args.steps,
        "steps_timed": len(ts),
        "warmup": n_warm,
        "ms_per_step": med * 1e3,
        "ms_per_step_mean": float(np.mean(ts)) * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c128 (f64 complex)",
        "data": "synthetic",
        "config": config,
        "cpu_baseline": {
            "value": value,
            "unit": "matvec/s",
            "cores": ncpu,
            "cpu_model": cpu_model(),
            "kind": kind,
            "sample": f"{len(ts)} full matvecs (median; bounded to ~60 s) after {n_warm} warm-up, {desc}, "
            f"workers=1, default BLAS threads ({ncpu})",
        },
        "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
