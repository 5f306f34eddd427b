"""Decode-round time of a workload's steady state with the library RT_LIB_PATH selects
(tools/ab_build.py): device time of K rounds between CUDA events on the engine stream.
Usage: ab_step.py [--workload C3] [--steps 20]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import profile_step  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    eng, now = profile_step.setup(None, workload=a.workload)
    for _ in range(3):
        eng.step(now())
    eng.sync()
    eng.mark(0)
    toks = 0
    for _ in range(a.steps):
        toks += eng.step(now())["n_running"]
    eng.mark(1)
    eng.sync()
    ms = eng.elapsed_ms() / a.steps
    print(f"{os.environ.get('RT_LIB_PATH', 'default')}: {a.workload} {ms:.3f} ms/step "
          f"{toks / a.steps / ms * 1e3:.0f} tok/s", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
