"""Probe: NN (MN-major B) tcgen05 GEMM against fp64 under descriptor variants (ENKS_TC_MN)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

ops = DeviceOps()
M, N, K = 128, 64, 32
g = torch.Generator().manual_seed(0)
A = torch.randn(M, K, generator=g)
B = torch.randn(K, N, generator=g)
bh, bl = ops.empty(K, N), ops.empty(K, N)
ops.tf32_split(B.cuda(), bh, bl)
ref = A.double() @ B.double()
for mode in ("0", "1", "2", "3"):
    os.environ["ENKS_TC_MN"] = mode
    C = ops.zeros(M, N)
    ops.gemm_nn_tc(A.cuda(), bh, bl, C, split=1)
    err = (C.double().cpu() - ref).abs()
    print("mode", mode, "maxerr", err.max().item(), "rows bad", int((err.max(1).values > 1e-3).sum()),
          "cols bad", int((err.max(0).values > 1e-3).sum()))
# identity B to see the column mapping
os.environ["ENKS_TC_MN"] = "0"
B = torch.zeros(K, N)
for k in range(K):
    B[k, k] = 1.0
ops.tf32_split(B.cuda(), bh, bl)
A = torch.arange(M * K, dtype=torch.float32).reshape(M, K) % 97
C = ops.zeros(M, N)
ops.gemm_nn_tc(A.cuda(), bh, bl, C, split=1)
c = C.cpu()
print("row0 of C (expect A[0,:32], zeros):", c[0, :40].tolist())
print("A row0:", A[0, :32].tolist())
