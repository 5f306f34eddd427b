"""Few-tile decode projections at N = 256 rows: CTA pairs over (m-pair, n-half) tiles with the
whole K range (no split-K exchange; the second n-half re-reads the weights from L2) against
the decode pair split-K kernel and cuBLAS.  Weights cycled through 8 copies (HBM)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tools"))
from proj_sweep import SHAPES, COPIES, timeit  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    for name in sys.argv[2:] or ["qkv", "o", "down"]:
        M, K = SHAPES[name]
        ws = [torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
              for _ in range(COPIES)]
        cap = ((N + 255) // 256) * 256
        X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(N, M, device="cuda")
        ref = None
        cells = []
        for label, path, bn in (("dec", 4, 0), ("pair128", 3, 128), ("pair256", 3, 256)):
            us = timeit(lambda i: rt.gemm_tiled(ws[i], X, out, M, N, K, cap, 0, path=path, bn=bn))
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            err = (out - ref).abs().max().item()
            cells.append(f"{label}:{us:6.1f}us(d={err:.1e})")
        Wr = [w[:M * K].view(M, K) for w in ws]
        us = timeit(lambda i: torch.nn.functional.linear(X[:N], Wr[i]))
        cells.append(f"cublas:{us:6.1f}")
        print(f"N={N} {name:5s} " + " ".join(cells), flush=True)


if __name__ == "__main__":
    main()
