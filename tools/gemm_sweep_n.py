import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo") + "/tools")
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import gemm_bench as g
for N in (64, 128, 192, 256, 320, 384, 512):
    row = []
    for name in ("qkv", "o", "gu", "down"):
        M, K = g.SHAPES[name]
        us, gbs = g.bench(M, K, N, 0, iters=30)
        tf = 2 * M * K * N / us / 1e6
        row.append(f"{name}:{us:7.1f}us {tf:5.0f}TF {gbs:5.0f}GB/s")
    print(N, " | ".join(row), flush=True)
