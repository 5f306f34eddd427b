"""Profile target: the bench's C2 engine configuration, setup + warmup outside the
profiler range, then `--steps` rounds inside cudaProfilerStart/Stop (use with
`ncu --profile-from-start off`)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def setup(B=None, flags=0, workload="C2", gemm_path=0):
    """The bench's steady state for a workload (bench.WORKLOADS: C2 / C3 / C4): its agents
    resident, decode-only rounds.  B overrides the agent count."""
    shape = MODEL_SHAPES["llama3-8b"]
    vocab = make_vocab(shape.vocab)
    wl = bench.WORKLOADS[workload]
    B = B or wl["agents"]
    max_ctx = wl["max_ctx"]
    n_pages = min(B * ((max_ctx + 15) // 16), 56 * 1024)
    p = engine_params("b200-roofline", max_batch=B, max_tasks=4 * B, max_ctx=max_ctx, n_pages=n_pages,
                      clock_mode=1)
    eng = rt.Engine(shape, p, vocab, seed=1234, flags=flags, max_rows_per_forward=8192, gemm_path=gemm_path)
    t0 = time.perf_counter()
    now = lambda: int((time.perf_counter() - t0) * 1e6)  # noqa: E731
    for j in range(B):
        tr = bench.agent_request(workload, vocab, j, 0, 0, plan_len=64)
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
    ap.add_argument("--agents", type=int, default=None)
    ap.add_argument("--workload", default="C3", choices=sorted(bench.WORKLOADS))
    a = ap.parse_args()
    eng, now = setup(a.agents, workload=a.workload)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        info = eng.step(now())
    eng.sync()
    torch.cuda.profiler.stop()
    print("profiled", a.steps, "steps at B =", info["n_running"], info)
    # algorithmic attention bytes of the last profiled round (per layer launch): decode row r
    # attends positions 0 .. pos_r -> K + V of every kv head, plus q and o
    rows = eng.dump(rt.RT_DUMP_ROWS, np.int32).reshape(-1, 3)
    s = eng.shape
    kv = int((rows[:, 1].astype(np.int64) + 1).sum()) * 2 * s.n_kv_heads * s.head_dim * 2
    qo = 2 * len(rows) * s.n_q_heads * s.head_dim * 2
    print(f"attention algorithmic bytes per layer launch: {kv + qo} ({len(rows)} rows, kv {kv}, q+o {qo})")


if __name__ == "__main__":
    main()
