"""Decode pair kernel (k_gemm_dec) at N rows: split-K count S over pairs (forced through
rt_op_gemm_tiled's splits argument), weights cycled through 8 copies.  Usage: dec_splits.py N"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402
from proj_sweep import SHAPES, COPIES, timeit  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    for name in ("qkv", "o", "down"):
        M, K = SHAPES[name]
        ws = [torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
              for _ in range(COPIES)]
        cap = ((N + 255) // 256) * 256
        X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(N, M, device="cuda")
        cells = []
        for S in (0, 2, 3, 4):
            us = timeit(lambda i: rt.gemm_tiled(ws[i], X, out, M, N, K, cap, S, path=4))
            cells.append(f"S{S or 'auto'}:{us:6.1f}")
        print(f"N={N} {name:5s} " + " ".join(cells), flush=True)


if __name__ == "__main__":
    main()
