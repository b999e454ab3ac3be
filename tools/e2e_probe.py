"""Diagnostics: where the end-to-end host-buffer matvec spends its time at a config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2405_15573_b200 import workloads
from paper_2405_15573_b200.device import DeviceOperator
from paper_2405_15573_b200.packer import pack

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
u = workloads.build_operator(cfg)
op = DeviceOperator(pack(u), device="cuda:0")
n = u.shape[1]
xh = torch.from_numpy(workloads.seeded_vector(n, 0)).pin_memory()
wh = torch.empty(n, dtype=torch.complex128).pin_memory()
xd = xh.cuda()
wd = torch.empty_like(xd)


def t(f, k=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / k * 1e6


print("h2d us", t(lambda: xd.copy_(xh, non_blocking=True)))
print("d2h us", t(lambda: wh.copy_(wd, non_blocking=True)))
print("h2d+d2h us", t(lambda: (xd.copy_(xh, non_blocking=True), wh.copy_(wd, non_blocking=True))))
print("kernel (device api) us", t(lambda: op.matvec(xd, out=wd)))
print("memset us", t(lambda: wd.zero_()))
print("e2e host api us", t(lambda: op.matvec_host(xh.numpy(), out=wh.numpy())))
print("sync-per-call device api us", t(lambda: (op.matvec(xd, out=wd), torch.cuda.synchronize())))
