"""Time the tcgen05 cross-moment GEMM alone: P (M x p) = A (M x K) Yc^T, per product mask."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 19200
K = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
N = 256
ops = DeviceOps()
A = torch.randn(M, K, device="cuda")
B = torch.randn(N, K, device="cuda")
bh, bl = torch.empty_like(B), torch.empty_like(B)
ops.tf32_split(B, bh, bl)
C = torch.empty(M, N, device="cuda")
for mask in ("7", "4", "1", "6"):
    os.environ["ENKS_TC_PRODUCTS"] = mask
    for _ in range(2):
        ops.gemm_nt_tc(A, bh, bl, C)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        ops.gemm_nt_tc(A, bh, bl, C)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"M={M} K={K} products={mask}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TF/s algorithmic, "
          f"A stream {M * K * 4 / ms / 1e6:.0f} GB/s")
