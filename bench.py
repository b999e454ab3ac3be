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
    ap.add_argument("--format", default="uh", choices=["uh", "h"],
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
    """The oracle port (restating uniform.py:476-556) on the host cores: best of BLAS threads
    {1, all}, bounded to ~sample_s seconds of CPU work."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from matvec_oracle import oracle_matvec_uh

    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    ncpu = os.cpu_count() or 1
    best = None
    for threads in sorted({1, ncpu}):
        ctx = threadpool_limits(limits=threads) if threadpool_limits else None
        try:
            oracle_matvec_uh(u, x)  # warm-up, excluded
            ts = []
            t_end = time.perf_counter() + sample_s / 2
            while len(ts) < 3 or (time.perf_counter() < t_end and len(ts) < 50):
                t0 = time.perf_counter()
                oracle_matvec_uh(u, x)
                ts.append(time.perf_counter() - t0)
        finally:
            if ctx is not None:
                ctx.__exit__(None, None, None)
        cand = (min(ts), threads, len(ts), float(np.median(ts)))
        if best is None or cand[0] < best[0]:
            best = cand
    t, threads, reps, med = best
    return {
        "value": 1.0 / t,
        "unit": "matvec/s",
        "cores": threads,
        "cpu_model": cpu_model(),
        "host_cpus": ncpu,
        "kind": "port",
        "sample": f"{reps} full matvecs (min of reps; median {med * 1e3:.1f} ms) after 1 warm-up, "
        f"oracle/matvec_oracle.py (restates uniform.py:476-556), BLAS threads best of {{1,{ncpu}}}",
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2405_15573_b200 import workloads

    if args.config == 5:
        if args.impl == "reference":
            run_reference(args, rank, world, {"workload": "cfg5_cfg3_operator_x_%d_rhs" % args.nrhs, "N": 81920,
                                              "nrhs": args.nrhs})
        else:
            run_multi_rhs(args, world, rank, local_rank)
        return
    meta = workloads.CONFIGS[args.config]
    config = {
        "workload": meta["name"],
        "N": meta["N"],
        "values": "seeded synthetic on the reference-built structure"
        + (" and ranks (rank-profile surrogate)" if meta["kind"] == "profile" else " (BASELINE config 4 spec)"),
        "vector": "default_rng(0) complex Gaussian, tree order",
        "mode": args.mode,
        "adjoint": bool(args.adjoint),
        "parallelism": f"row-partition x{args.gpus}" if args.gpus > 1 else "single GPU",
    }
    if args.emulate_ranks > 1:
        config["parallelism"] = (f"peer-exchange partition of {args.emulate_ranks} ranks emulated in one launch "
                                 f"on one GPU (1/{args.emulate_ranks} of the SMs each)")

    if args.impl == "reference":
        run_reference(args, rank, world, config)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)

    t_build = time.perf_counter()
    u = workloads.build_operator(args.config) if args.format == "uh" else workloads.build_h_operator(args.config)
    if args.format == "h":
        config["format"] = "H-matrix (matvec_h, hmatrix.py:143-184), ranks of the reference's assemble_h"
    if args.view != "full":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from matvec_oracle import farfield_only, nearfield_only

        u = farfield_only(u) if args.view == "far" else nearfield_only(u)
        config["view"] = args.view
    x_np = workloads.seeded_vector(u.shape[1], 0)
    from paper_2405_15573_b200.packer import pack

    if world > 1:
        from paper_2405_15573_b200.dist import DistributedOperator

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
        else:
            packed = pack(u)
        op = DeviceOperator(packed, device=dev)
    t_build = time.perf_counter() - t_build

    n_in = u.shape[0] if args.adjoint else u.shape[1]
    x = torch.from_numpy(x_np if not args.adjoint else workloads.seeded_vector(n_in, 0)).to(dev)
    stream = torch.cuda.current_stream(dev)

    def step(out=None):
        return op.matvec(x, adjoint=args.adjoint, mode=args.mode, out=out)

    out = step()
    # L2 policy: operator bytes vs the 126 MB L2
    full_bytes = workloads.algorithmic_bytes(packed)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = full_bytes / max(world, 1) < 4 * l2_bytes and args.l2 == "auto"
    flush_buf = torch.empty(int(2 * l2_bytes) // 4 + 1024, dtype=torch.float32, device=dev) if flush else None
    flush_rd = torch.zeros(int(2 * l2_bytes) // 4 + 1024, dtype=torch.float32, device=dev) if flush else None

    def flush_l2():
        # write a buffer > L2, then read another one: the read evicts the dirty lines (their
        # write-back happens here, untimed) and leaves L2 cold and clean for the timed step
        flush_buf.zero_()
        flush_rd.sum()

    config["l2"] = (
        f"L2 flushed between steps ({flush_buf.numel() * 4 / 1e6:.0f} MB write + read, untimed)" if flush
        else (f"L2-hot: no flush (operator {full_bytes / 1e6:.0f} MB, L2 {l2_bytes / 1e6:.0f} MB)" if args.l2 == "hot"
              else f"operator {full_bytes / max(world, 1) / 1e9:.2f} GB per GPU >> L2 {l2_bytes / 1e6:.0f} MB, no flush")
    )
    for _ in range(max(args.warmup, 3)):
        if flush:
            flush_l2()
        step(out)
    torch.cuda.synchronize(dev)

    # timed region: events around every step's kernel(s) on the launching stream
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        if flush:
            flush_l2()
        starts[i].record(stream)
        step(out)
        ends[i].record(stream)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    per_step = np.array([s.elapsed_time(e) for s, e in zip(starts, ends)]) * 1e-3  # s
    kernel_s = float(per_step.mean())
    if world > 1:
        t = torch.tensor([kernel_s, float(np.median(per_step))], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        kernel_s, med_s = float(t[0]), float(t[1])
    else:
        med_s = float(np.median(per_step))

    # end to end through the reference-facing C-ABI call with host buffers (multi-GPU: the
    # same call gathers the output slices; time = max over ranks)
    e2e = None
    if True:
        xh = torch.from_numpy(x.cpu().numpy()).pin_memory()
        wh = torch.empty(u.shape[1 if args.adjoint else 0], dtype=torch.complex128).pin_memory()
        xh_np, wh_np = xh.numpy(), wh.numpy()
        for _ in range(10):  # includes the host-I/O vs copy-path choice (4 calls each)
            op.matvec_host(xh_np, adjoint=args.adjoint, out=wh_np, mode=args.mode)
        k_e2e = max(10, min(args.steps, 200))
        if world > 1:
            torch.distributed.barrier()
        te = time.perf_counter()
        for _ in range(k_e2e):
            op.matvec_host(xh_np, adjoint=args.adjoint, out=wh_np, mode=args.mode)
        te = (time.perf_counter() - te) / k_e2e
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {
            "value": 1.0 / te,
            "unit": "matvec/s",
            "h2d_bytes_per_step": int(16 * n_in),
            "d2h_bytes_per_step": int(16 * (u.shape[1] if args.adjoint else u.shape[0])),
            "api": "uhmv_matvec_host (C ABI, pinned host x/w, H2D + kernels + D2H + sync, wall clock)",
        }
        choice = op.host_io_choice(args.adjoint) if hasattr(op, "host_io_choice") else None
        if choice is not None:
            e2e["path"] = ("host-I/O launch: x read over PCIe by the P1 ops, finished output leaves drained "
                           "to the pinned host buffer inside the kernel" if choice
                           else "H2D copy + launch + D2H copy (faster than the host-I/O launch here)")

    peak, peak_kind = measured_peaks()
    alg_bytes_total = workloads.algorithmic_bytes(packed)
    value = 1.0 / kernel_s
    achieved = alg_bytes_total / world / kernel_s / 1e9  # per GPU
    traffic = load_traffic(args.config)
    roofline = {
        "bound": "hbm",
        "achieved": achieved,
        "peak": peak,
        "unit": "GB/s",
        "frac": achieved / peak,
        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
        "frac_vs_8000_nominal": achieved / 8000.0,
        "traffic": traffic,
        "algorithmic_bytes_per_launch": int(alg_bytes_total / world),
        "kernel": "bulk::uhmv_bulk_peer_kernel" if (args.emulate_ranks > 1 or getattr(op, "exchange", "") == "peer") else
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
        "warmup": max(args.warmup, 3),
        "ms_per_step": kernel_s * 1e3,
        "ms_per_step_median": med_s * 1e3,
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


def dmma_peak(device_index: int):
    import ctypes

    from paper_2405_15573_b200 import _lib

    pk = ctypes.c_double()
    _lib.check(_lib.lib().uhmv_dmma_peak(device_index, ctypes.byref(pk)), "uhmv_dmma_peak")
    return pk.value


def run_multi_rhs(args, world, rank, local_rank):
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
    steps = max(3, min(args.steps, 50))
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
    t = float(np.mean([a.elapsed_time(b) for a, b in ev])) * 1e-3
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
        "config": {"workload": "cfg5_cfg3_operator_x_%d_rhs" % R, "N": n, "nrhs": R,
                   "parallelism": (f"{world} GPUs, each its own block of {R} right-hand sides (no exchange)"
                                   if world > 1 else "single GPU"),
                   "values": "seeded synthetic on the reference-built cfg3 structure and ranks"},
        "roofline": {"bound": "tensor", "achieved": flops / t / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": flops / t / 1e12 / peak,
                     "peak_source": "uhmv_dmma_peak: measured DMMA m16n8k16 f64 throughput on this GPU",
                     "traffic": None, "flops_per_launch": flops, "kernel": "mrtc::uhmv_mrtc_kernel"},
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
    v = d.get(f"cfg{cfg}")
    return float(v) if v is not None else None


def run_reference(args, rank, world, config):
    """--impl reference: the reference algorithm (oracle port of uniform.py:476-556) on the
    host CPU, all host threads; rank 0 only under torchrun."""
    if rank != 0:
        return
    from paper_2405_15573_b200 import workloads

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from matvec_oracle import oracle_matvec_uh

    cfg = 3 if args.config == 5 else args.config  # config 5 = the config-3 operator, column loop
    u = workloads.build_operator(cfg)
    n_in = u.shape[0] if args.adjoint else u.shape[1]
    if args.config == 5:  # the reference has no block product: one matvec per right-hand side
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n_in, args.nrhs)) + 1j * rng.standard_normal((n_in, args.nrhs))
    else:
        X = workloads.seeded_vector(n_in, 0)[:, None]
    n_warm = max(1, min(args.warmup, 3))  # untimed warm-up matvecs (bounded too)
    for i in range(n_warm):
        oracle_matvec_uh(u, X[:, i % X.shape[1]], adjoint=args.adjoint)
    # bounded sample: the timed steps stop after ~60 s of CPU work (a step = one matvec; for
    # config 5 one right-hand side of the block, the metric being right-hand sides per second)
    ts = []
    t_all = time.perf_counter()
    for i in range(max(args.steps, 1)):
        t0 = time.perf_counter()
        oracle_matvec_uh(u, X[:, i % X.shape[1]], adjoint=args.adjoint)
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > 60.0:
            break
    mean = float(np.mean(ts))
    value = 1.0 / mean
    ncpu = os.cpu_count() or 1
    line = {
        "impl": "reference",
        "metric": ("uniform-H matvecs/sec (multi-RHS block, config 5)" if args.config == 5
                   else "uniform-H matvecs/sec (effective HBM GB/s, roofline fraction)"),
        "value": value,
        "unit": "matvec/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": n_warm,
        "ms_per_step": mean * 1e3,
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
            "kind": "port",
            "sample": f"{len(ts)} full matvecs (bounded to ~60 s), oracle/matvec_oracle.py (restates "
            f"uniform.py:476-556), default BLAS threads ({ncpu}); the Python reference itself cannot "
            "travel to the GPU box",
        },
        "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
