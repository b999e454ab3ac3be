"""Diagnostics: op timeline of one profiled bulk matvec (usage: python tools/timeline.py CFG
[fwd|adj] [full|far|near] [uh|h]).  Prints, per op kind, when its ops start / get their
dependencies / end, how long they wait for dependencies vs compute, and the kernel span;
saves the raw timeline to gpurun_out/timeline_cfgN.npz."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch

from paper_2405_15573_b200 import workloads
from paper_2405_15573_b200.device import DeviceOperator
from paper_2405_15573_b200.packer import KIND_NAMES, pack

cfg = int(sys.argv[1])
adj = len(sys.argv) > 2 and sys.argv[2] == "adj"
view = sys.argv[3] if len(sys.argv) > 3 else "full"
fmt = sys.argv[4] if len(sys.argv) > 4 else "uh"
u = {"uh": workloads.build_operator, "h": workloads.build_h_operator,
     "sym": workloads.build_symmetric_operator}[fmt](cfg)
if view != "full":
    from matvec_oracle import farfield_only, nearfield_only

    u = farfield_only(u) if view == "far" else nearfield_only(u)
if fmt == "h":
    from paper_2405_15573_b200.packer_h import pack_h

    op = DeviceOperator(pack_h(u), device="cuda:0")
elif fmt == "sym":
    from paper_2405_15573_b200.packer_sym import pack_sym

    op = DeviceOperator(pack_sym(u), device="cuda:0")
else:
    op = DeviceOperator(pack(u), device="cuda:0")
x = torch.from_numpy(workloads.seeded_vector(u.shape[0] if adj else u.shape[1], 0)).cuda()
for _ in range(3):
    op.matvec(x, adjoint=adj)
t, kinds = op.trace(adjoint=adj, x=x)
prog = op.progs[1] if adj else op.progs[0]
ticket = np.empty(prog.n_ops, dtype=np.int64)
ticket[prog.fused_order] = np.arange(prog.n_ops)
span = t[:, 2].max()
print(f"cfg{cfg} {fmt} {'adj' if adj else 'fwd'} {view}: span {span / 1e3:.1f} us, ops {prog.n_ops}")
for k in range(7):
    m = kinds == k
    if not m.any():
        continue
    st, dr, en = t[m, 0], t[m, 1], t[m, 2]
    print(f"  {KIND_NAMES[k]:5s} n {m.sum():5d}  start {st.min()/1e3:6.1f}-{st.max()/1e3:6.1f}  "
          f"deps-met {np.median(dr)/1e3:6.1f} (max {dr.max()/1e3:6.1f})  end {np.median(en)/1e3:6.1f} (max {en.max()/1e3:6.1f})  "
          f"wait {np.mean(dr - st)/1e3:5.2f}  run {np.mean(en - dr)/1e3:5.2f} (max {np.max(en - dr)/1e3:5.2f}) us")
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/timeline_cfg{cfg}_{'adj' if adj else 'fwd'}_{view}.npz", t=t, kinds=kinds, ticket=ticket,
         waits=prog.waits, ops=prog.ops, sigs=prog.sigs)
