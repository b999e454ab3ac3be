"""Diagnostics: multi-RHS host-buffer pipeline at config 3 (chunk sizes, device-only times)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2405_15573_b200 import workloads
from paper_2405_15573_b200.device import DeviceOperator
from paper_2405_15573_b200.packer import pack

u = workloads.build_operator(3)
op = DeviceOperator(pack(u), device="cuda:0")
n = u.shape[1]
rng = np.random.default_rng(0)
Xh = torch.from_numpy(rng.standard_normal((n, 64)) + 1j * rng.standard_normal((n, 64))).pin_memory()
Wh = torch.empty((n, 64), dtype=torch.complex128).pin_memory()


def t(f, k=5):
    f()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / k * 1e3


for R in (16, 32, 64):
    X = Xh[:, :R].contiguous().cuda()
    print("device matmat R=%d: %.3f ms" % (R, t(lambda: op.matmat(X))))
for chunk in (16, 32, 64):
    print("matmat_host chunk=%d: %.3f ms" % (chunk, t(lambda: op.matmat_host(Xh.numpy(), out=Wh.numpy(), chunk=chunk))))
Xd = torch.empty((n, 64), dtype=torch.complex128, device="cuda:0")
print("contiguous H2D 84 MB: %.3f ms" % t(lambda: Xd.copy_(Xh, non_blocking=True)))
