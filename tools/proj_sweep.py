"""Sweep of the single-CTA decode projection kernel (k_gemm_tc) over tile width BN and
cluster split-K S at fixed N rows, weights cycled through 8 copies (every launch streams
from HBM).  Usage: proj_sweep.py N [shape ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)}
COPIES = 8


def timeit(fn, it=32):
    for i in range(COPIES):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(it):
        fn(i % COPIES)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    names = sys.argv[2:] or list(SHAPES)
    for name in names:
        M, K = SHAPES[name]
        ws = [torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
              for _ in range(COPIES)]
        cap = ((N + 255) // 256) * 256
        X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(N, M, device="cuda")
        cells = []
        for bn in (64, 128, 256):
            for S in (1, 2, 3, 4, 6, 8):
                tiles = ((M + 127) // 128) * ((N + bn - 1) // bn)
                if S > 1 and tiles * S > (296 if bn <= 128 else 148):
                    continue
                try:
                    us = timeit(lambda i: rt.gemm_tiled(ws[i], X, out, M, N, K, cap, S, path=1, bn=bn))
                    cells.append(f"bn{bn}/S{S}:{us:6.1f}")
                except Exception as ex:  # noqa: BLE001
                    cells.append(f"bn{bn}/S{S}:ERR")
        us = timeit(lambda i: rt.gemm_tiled(ws[i], X, out, M, N, K, cap, 0))
        cells.append(f"auto:{us:6.1f}")
        print(f"N={N} {name:5s} " + " ".join(cells), flush=True)


if __name__ == "__main__":
    main()
