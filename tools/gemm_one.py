"""One projection shape, `--iters` back-to-back launches after 3 warm-ups (ncu target)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--splits", type=int, default=8)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    W = (torch.randn(a.M, a.K, device="cuda") * 0.02).to(torch.bfloat16)
    Wt = torch.empty(((a.M + 127) // 128) * 128 * a.K, dtype=torch.bfloat16, device="cuda")
    rt.pack_tiled(W, Wt, a.M, a.K)
    cap = ((a.N + 255) // 256) * 256
    X = torch.randn(cap, a.K, device="cuda").to(torch.bfloat16)
    out = torch.empty(a.N, a.M, device="cuda")
    for _ in range(3 + a.iters):
        rt.gemm_tiled(Wt, X, out, a.M, a.N, a.K, cap, a.splits)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
