"""Time the fp16-pair cross-moment contraction at C3 shapes vs the 3xTF32 kernel."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

ops = DeviceOps()
for M in (2560, 8064, 19200):
    K, N = 131072, 256
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    ah = torch.empty(M, K, dtype=torch.float16, device="cuda"); al = torch.empty_like(ah)
    bh = torch.empty(N, K, dtype=torch.float16, device="cuda"); bl = torch.empty_like(bh)
    sa, sb = torch.empty(M, device="cuda"), torch.empty(N, device="cuda")
    ops.f16pair_split(A, ah, al, sa)
    ops.f16pair_split(B, bh, bl, sb)
    C = torch.empty(M, N, device="cuda")
    for chain in ("3", "2"):
        os.environ["ENKS_F16P_PRODUCTS"] = chain
        for _ in range(2):
            ops.gemm_f16pair(ah, al, sa, bh, bl, sb, C)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            ops.gemm_f16pair(ah, al, sa, bh, bl, sb, C)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        print(f"f16pair pair={os.environ.get('ENKS_F16P_PAIR', '1')} M={M} products={chain}: {ms:.3f} ms {2 * M * N * K / ms / 1e9:.0f} TF/s "
              f"A {M * K * 4 / ms / 1e6:.0f} GB/s", flush=True)
    del A, ah, al
