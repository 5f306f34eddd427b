"""Prefill projection time vs rows N with the engine's dispatch (`python tools/gemm_policy_sweep.py
[names]` prints one line per N; forced paths: tools/proj_bench.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gemm_bench as g  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["gu", "qkv", "o", "down"]
for N in range(160, 1025, 32):
    row = []
    for name in names:
        M, K = g.SHAPES[name]
        us, _ = g.bench(M, K, N, 0, iters=20)
        row.append(f"{name} {us:7.1f}")
    print(N, " | ".join(row), flush=True)
