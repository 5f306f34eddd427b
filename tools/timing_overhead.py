import os, sys, time
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"]); sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"] + "/tools")
import torch, profile_step
from paper_2412_18695_b200 import rt
for flags in (rt.RT_FLAG_TIMING, 0, rt.RT_FLAG_TIMING, 0):
    eng, now = profile_step.setup(64, flags=flags)
    for _ in range(5): eng.step(now())
    eng.sync(); eng.mark(0)
    for _ in range(20): eng.step(now())
    eng.mark(1); ms = eng.elapsed_ms()
    print("flags", flags, "ms/step", round(ms / 20, 3), "tok/s", round(64 * 20 / ms * 1e3))
    eng.close()
