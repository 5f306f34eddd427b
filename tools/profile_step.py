"""Profile target: the bench's C2 engine configuration, setup + warmup outside the
profiler range, then `--steps` rounds inside cudaProfilerStart/Stop (use with
`ncu --profile-from-start off`)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import bench  # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params  # noqa: E402
from synth.traces import make_trace  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def setup(B, flags=0, config="c2"):
    """The bench's steady state: B agents resident, decode-only rounds.  config "c2": drone
    agents (prompt 1300); "c3": half drone, half robot arm (prompt 2884), SURVEY §8(d) C3."""
    shape = MODEL_SHAPES["llama3-8b"]
    vocab = make_vocab(shape.vocab)
    max_ctx = bench.MAX_CTX if config == "c2" else 4096
    n_pages = B * 3 * ((max_ctx + 15) // 16) // 4 + 64
    p = engine_params("b200-roofline", max_batch=B, max_tasks=4 * B, max_ctx=max_ctx, n_pages=n_pages,
                      clock_mode=1)
    eng = rt.Engine(shape, p, vocab, seed=1234, flags=flags, max_rows_per_forward=8192)
    t0 = time.perf_counter()
    now = lambda: int((time.perf_counter() - t0) * 1e6)  # noqa: E731
    for j in range(B):
        if config == "c2" or j % 2 == 0:
            tr = bench.drone_request(vocab, j, 0, 0, plan_len=64)
        else:
            tr = make_trace(9 + (j // 2) % 3, vocab, seed=j, plan_len=64)
        eng.submit(j, tr.prompt, now(), tr.ert_us, tr.alpha, tr.beta, p.g_us, script=tr.plan)
    for _ in range(400):
        info = eng.step(now())
        if info["n_running"] == B and info["n_prefill_rows"] == 0:
            break
    for _ in range(50):   # WCET speed window forgets the prefill round; all B back in the batch
        info = eng.step(now())
        if info["n_running"] == B:
            break
    for _ in range(6):
        info = eng.step(now())
    eng.sync()
    return eng, now


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--agents", type=int, default=bench.AGENTS_PER_GPU)
    a = ap.parse_args()
    eng, now = setup(a.agents)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        info = eng.step(now())
    eng.sync()
    torch.cuda.profiler.stop()
    print("profiled", a.steps, "steps at B =", info["n_running"], info)


if __name__ == "__main__":
    main()
