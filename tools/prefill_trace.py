"""Kernel timeline of prefill rounds (k = 0 admissions of drone prompts), device trace."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import time  # noqa: E402
import bench  # noqa: E402
import trace_step  # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    shape = MODEL_SHAPES["llama3-8b"]
    vocab = make_vocab(shape.vocab)
    B = 64
    max_ctx = bench.WORKLOADS["C2"]["max_ctx"]
    n_pages = B * 3 * ((max_ctx + 15) // 16) // 2
    p = engine_params("b200-roofline", max_batch=B, max_tasks=4 * B, max_ctx=max_ctx, n_pages=n_pages,
                      clock_mode=1)
    eng = rt.Engine(shape, p, vocab, seed=1234, flags=rt.RT_FLAG_TRACE | rt.RT_FLAG_TIMING,
                    max_rows_per_forward=8192)
    t0 = time.perf_counter()
    now = lambda: int((time.perf_counter() - t0) * 1e6)  # noqa: E731
    for rep in range(a.reps + 1):
        for j in range(a.requests):
            tr = bench.agent_request("C2", vocab, j + 100 * rep, 0, 0, plan_len=4)
            eng.submit(j, tr.prompt, now(), tr.ert_us, tr.alpha, tr.beta, p.g_us, script=tr.plan)
        eng.sync()
        eng.reset_stats()
        info = eng.step(now())
        eng.sync()
        if rep == 0:
            continue
        tr_ = eng.trace()
        agg, span, n, _ = trace_step.analyse(tr_)
        print(f"prefill round: {info['n_prefill_rows']} prefill rows, {info['n_rows']} rows, span {span:.0f} us")
        for name, (cnt, lead, gap, body, ctas, _m, _e) in sorted(agg.items(), key=lambda x: -(x[1][2] + x[1][3]))[:8]:
            print(f"   {name:28s} n={cnt:4d} body/launch {body / cnt:9.1f} us  total {gap + body:9.1f} us")
        for _ in range(8):   # drain: finish the short plans
            eng.step(now())
        eng.poll()
    eng.close()


if __name__ == "__main__":
    main()
