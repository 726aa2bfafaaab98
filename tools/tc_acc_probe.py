"""Probe: accuracy of the tcgen05 3xTF32 contraction per product set (ENKS_TC_PRODUCTS)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

ops = DeviceOps()
for K in (128, 4096):
    g = torch.Generator().manual_seed(1)
    A = torch.randn(128, K, generator=g) + 0.5
    B = torch.randn(256, K, generator=g)
    dA, dB = A.cuda(), B.cuda()
    bh, bl = ops.empty(256, K), ops.empty(256, K)
    ops.tf32_split(dB, bh, bl)
    ref = A.double() @ B.double().t()
    scale = A.double().abs() @ B.double().abs().t()
    for mode in (4, 5, 6, 7):
        os.environ["ENKS_TC_PRODUCTS"] = str(mode)
        C = ops.zeros(128, 256)
        ops.gemm_nt_tc(dA, bh, bl, C, split=1)
        print(K, mode, ((C.double().cpu() - ref).abs() / scale).max().item())
    ah, al = ops.empty(128, K), ops.empty(128, K)
    ops.tf32_split(dA, ah, al)
    r1 = ah.double().cpu() @ bh.double().cpu().t()
    print(K, "emul 1xtf32", ((r1 - ref).abs() / scale).max().item())
    r3 = r1 + al.double().cpu() @ bh.double().cpu().t() + ah.double().cpu() @ bl.double().cpu().t()
    print(K, "emul 3xtf32", ((r3 - ref).abs() / scale).max().item())

# short accumulation chains: split-K so each CTA accumulates only `cps` chunks in TMEM
K = 4096
g = torch.Generator().manual_seed(1)
A = torch.randn(128, K, generator=g) + 0.5
B = torch.randn(256, K, generator=g)
dA, dB = A.cuda(), B.cuda()
bh, bl = ops.empty(256, K), ops.empty(256, K)
ops.tf32_split(dB, bh, bl)
ref = A.double() @ B.double().t()
scale = A.double().abs() @ B.double().abs().t()
os.environ["ENKS_TC_PRODUCTS"] = "7"
for split in (1, 4, 16, 32, 128):
    C = ops.zeros(128, 256)
    ops.gemm_nt_tc(dA, bh, bl, C, split=split)
    print("split", split, "chain K", K // split, ((C.double().cpu() - ref).abs() / scale).max().item())
