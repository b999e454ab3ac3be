"""Quick multi-RHS timing probe (config 5 = config 3 operator x 64 RHS) on the GPU box."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from matvec_oracle import oracle_matvec_uh  # noqa: E402
from paper_2405_15573_b200 import workloads  # noqa: E402
from paper_2405_15573_b200.device import DeviceOperator  # noqa: E402
from paper_2405_15573_b200.packer import pack  # noqa: E402

import ctypes  # noqa: E402

from paper_2405_15573_b200 import _lib  # noqa: E402

pk = ctypes.c_double()
_lib.check(_lib.lib().uhmv_dmma_peak(0, ctypes.byref(pk)), "dmma_peak")
print(f"measured DMMA peak: {pk.value:.2f} TFLOP/s")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
R = int(sys.argv[2]) if len(sys.argv) > 2 else 64
u = workloads.build_operator(cfg)
dop = DeviceOperator(pack(u), device="cuda:0")
rng = np.random.default_rng(0)
n = u.shape[1]
X = rng.standard_normal((n, R)) + 1j * rng.standard_normal((n, R))
Xd = torch.from_numpy(X).cuda()
W = dop.matmat(Xd)
torch.cuda.synchronize()
ref0 = oracle_matvec_uh(u, X[:, 0])
ref7 = oracle_matvec_uh(u, X[:, R - 1])
Wc = W.cpu().numpy()
print("rel col0", np.linalg.norm(Wc[:, 0] - ref0) / np.linalg.norm(ref0),
      "col-1", np.linalg.norm(Wc[:, -1] - ref7) / np.linalg.norm(ref7))
for _ in range(3):
    dop.matmat(Xd)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
K = 10
for _ in range(K):
    dop.matmat(Xd)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / K
p = dop.packed
flops = 8 * R * p.bytes_alg / 16
print(f"cfg{cfg} R={R}: {ms:.3f} ms per block, {R / ms * 1e3:.0f} matvec/s, "
      f"{flops / ms / 1e9:.2f} TFLOP/s (8 flop per complex MAC), single-RHS ms {0}")
