"""Bottleneck probe for the tcgen05 contraction: debug knobs x cluster size x products."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

M, K, N = 19200, 131072, 256
ops = DeviceOps()
A = torch.randn(M, K, device="cuda")
B = torch.randn(N, K, device="cuda")
bh, bl = torch.empty_like(B), torch.empty_like(B)
ops.tf32_split(B, bh, bl)
C = torch.empty(M, N, device="cuda")


def run(tag):
    for _ in range(2):
        ops.gemm_nt_tc(A, bh, bl, C)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        ops.gemm_nt_tc(A, bh, bl, C)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    print(f"{tag:40s} {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.0f} TF/s  A {M * K * 4 / ms / 1e6:.0f} GB/s", flush=True)


for chain in ("4", "8", "16", "64", "100000"):
    for prod in ("7", "4"):
        os.environ.update(ENKS_TC_CHAIN=chain, ENKS_TC_PRODUCTS=prod)
        run(f"chain={chain} products={prod}")
os.environ.update(ENKS_TC_CHAIN="8", ENKS_TC_PRODUCTS="7")
