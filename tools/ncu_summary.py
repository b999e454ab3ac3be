"""Summarise an ncu report (run here, no GPU needed) into profiles/: key DRAM/roofline counters,
stall mix, and the per-launch list.  usage: python tools/ncu_summary.py REP.ncu-rep OUT.json [cfg]"""

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
    # FP64 tensor pipe (DMMA) of the multi-RHS engine (names from ncu --query-metrics --chip gb100)
    "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, r)}
        kernels.append(d)
    return kernels


def main():
    rep, out = sys.argv[1], sys.argv[2]
    cfg = sys.argv[3] if len(sys.argv) > 3 else None
    res = []
    for d in raw(rep):
        k = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
        for key in KEYS:
            if key in d:
                v, u = d[key]
                try:
                    k[key] = float(v.replace(",", ""))
                except ValueError:
                    k[key] = v
                k[key + ".unit"] = u
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[0] or 0)
                  for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        k["stall_mix_pct"] = {s: round(100 * v / tot, 1) for s, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        res.append(k)
    with open(out, "w") as fh:
        json.dump({"report": rep, "config": cfg, "kernels": res}, fh, indent=1)
    for k in res:
        print(json.dumps({x: k.get(x) for x in ("kernel", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum")}))


if __name__ == "__main__":
    main()
