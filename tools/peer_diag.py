"""Diagnostics: consecutive peer-emulation matvecs at a config, checked against the
single-GPU engine after every epoch (usage: python tools/peer_diag.py CFG WORLD [N])."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2405_15573_b200 import workloads
from paper_2405_15573_b200.device import DeviceOperator
from paper_2405_15573_b200.dist import PeerEmulation
from paper_2405_15573_b200.packer import pack

cfg, world = int(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
u = workloads.build_operator(cfg)
x = torch.from_numpy(workloads.seeded_vector(u.shape[1], 0)).cuda()
one = DeviceOperator(pack(u), device="cuda:0")
ref = one.matvec(x)
em = PeerEmulation(u, world, device="cuda:0")
import ctypes
from paper_2405_15573_b200 import _lib
diag = torch.zeros(512, dtype=torch.int64).view(torch.int32)[:512].pin_memory() if False else torch.zeros(512, dtype=torch.int32).pin_memory()
_lib.lib().uhmv_peer_set_diag(ctypes.c_void_p(diag.data_ptr()), int(os.environ.get("SPIN_LOG2", "22")))
out = torch.empty_like(ref)
for i in range(n):
    mode = i % 3
    sc = 1.0 + 0.37j * (i % 5)  # a different x each epoch: stale exchange data would show
    xs = x * sc
    ref = one.matvec(xs)
    t = time.time()
    if mode == 0:
        w = em.matvec(xs, out=out)
    elif mode == 1:
        w = em.matvec(xs.clone())
    else:
        w = torch.from_numpy(em.matvec_host(xs.cpu().numpy())).cuda()
    try:
        torch.cuda.synchronize()
    except Exception as e:
        d = diag.tolist()
        print("FAILED at", i, em.epoch, "n", d[0], flush=True)
        for k in range(min(d[0], 63)):
            print("  rec", d[8 + 8 * k: 16 + 8 * k], flush=True)
        raise
    err = (torch.linalg.norm(w - ref) / torch.linalg.norm(ref)).item()
    print(i, mode, "%.2e" % err, "%.1f ms" % ((time.time() - t) * 1e3), em.epoch, flush=True)
print("ok")
