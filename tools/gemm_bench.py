"""Microbenchmark of the tcgen05 projection kernel on the decode shapes (pre-packed
weights, CUDA events over many back-to-back launches)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336),
          "lm": (128256, 4096)}


def bench(M, K, N, splits, iters=50):
    W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.bfloat16)
    Wt = torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda")
    rt.pack_tiled(W, Wt, M, K)
    cap = ((N + 255) // 256) * 256
    X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(N, M, device="cuda")
    for _ in range(3):
        rt.gemm_tiled(Wt, X, out, M, N, K, cap, splits)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        rt.gemm_tiled(Wt, X, out, M, N, K, cap, splits)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    return us, M * K * 2 / us / 1e3


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    for name, (M, K) in SHAPES.items():
        res = []
        for s in [0, 1, 2, 3, 4, 5, 6, 8, 9, 12, 16]:
            if s > K // 64:
                continue
            try:
                us, gbs = bench(M, K, N, s)
                res.append(f"s{s}:{us:6.1f}us/{gbs:5.0f}")
            except Exception as ex:  # noqa: BLE001
                res.append(f"s{s}:ERR {ex}")
        print(name, M, K, " ".join(res), flush=True)
    print("auto splits (s0) per shape above; N =", N)
    # reference: a plain device copy of the same bytes
    for name, (M, K) in SHAPES.items():
        a = torch.empty(M * K, dtype=torch.bfloat16, device="cuda")
        b = torch.empty_like(a)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        for _ in range(3):
            b.copy_(a)
        e0.record()
        for _ in range(20):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"copy {name}: {us:6.1f} us  read+write {2 * M * K * 2 / us / 1e3:5.0f} GB/s")


if __name__ == "__main__":
    main()
