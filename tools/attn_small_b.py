import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"] + "/tools"); sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import attn_bench as A
for B, ctx in [(8, 1310), (8, 2884), (8, 8192), (16, 2884), (16, 8192), (32, 1310)]:
    us, gbs = A.bench(B, ctx)
    print(B, ctx, round(us, 1), round(gbs))
