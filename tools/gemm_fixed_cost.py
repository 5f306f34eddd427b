import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
from paper_2412_18695_b200 import rt
from proj_sweep import COPIES, timeit
for (M, K, N, path) in [(6144, 512, 256, 4), (6144, 1024, 256, 4), (6144, 4096, 256, 4), (4096, 512, 256, 4), (6144, 512, 64, 1), (6144, 4096, 64, 1), (4096, 512, 64, 1)]:
    ws = [torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02) for _ in range(COPIES)]
    cap = 256
    X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(N, M, device="cuda")
    us = timeit(lambda i: rt.gemm_tiled(ws[i], X, out, M, N, K, cap, 0, path=path))
    print(f"M={M} K={K} N={N} path={path}: {us:.1f} us  ({M*K*2/us/1e3:.0f} GB/s)")
