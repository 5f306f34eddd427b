"""Round structure of the CTA-pair projection kernel (k_gemm_2sm, forced pair path): time per
launch at N rows, K = 4096, for M = 256 x {pair-tiles}, weights cycled through 8 copies (every
launch streams from HBM).  One round = 74 co-resident pairs; gate/up at 256 rows is 112
pair-tiles (1.5 rounds).  Usage: pair_rounds.py [N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    K = 4096
    cap = ((N + 255) // 256) * 256
    X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
    for PT in (18, 37, 56, 74, 93, 112, 130, 148, 186, 222):
        M = 256 * PT
        ws = [torch.empty(M * K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02) for _ in range(8)]
        out = torch.empty(N, M, device="cuda")
        for w in ws:
            rt.gemm_tiled(w, X, out, M, N, K, cap, 0, path=3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        it = 32
        e0.record()
        for i in range(it):
            rt.gemm_tiled(ws[i % 8], X, out, M, N, K, cap, 0, path=3)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / it * 1e3
        print(f"N={N} pair-tiles {PT:4d} ({PT / 74:4.2f} rounds): {us:7.1f} us, {2 * M * N * K / us / 1e6:6.0f} TFLOP/s, "
              f"weights {M * K * 2 / us / 1e3:5.0f} GB/s", flush=True)
        del ws, out


if __name__ == "__main__":
    main()
