"""Launch each decoder projection once at N rows (after one warm-up launch) for an ncu capture
of the prefill-shaped projections: `ncu --kernel-name regex:k_gemm ... python tools/gemm_once.py 384`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gemm_bench as g  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 384
for name in ("qkv", "o", "gu", "down"):
    M, K = g.SHAPES[name]
    g.bench(M, K, N, 0, iters=1)
