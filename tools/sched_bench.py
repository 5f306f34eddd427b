"""Scheduling overhead vs queue size — the B200 analog of tab:sched_overhead (PAPER.md:739-752:
0.58 / 0.83 / 1.25 / 1.58 / 2.03 ms for 1 / 2 / 4 / 6 / 8 tasks, Python PriorityQueue).

Device time of k_sched_pre (ingest + Eq. 4 for every waiting task + sort + admission + paging
+ batch assembly) and k_sched_post (stop checker + retire + segment records) per round, CUDA
events, scheduling-only engine (RT_FLAG_NO_MODEL), max_batch 1 so N-1 tasks stay queued."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from synth import make_vocab, engine_params  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def run(n_tasks, rounds=200, trace=False):
    v = make_vocab(512)
    p = engine_params("b200-roofline", max_batch=1, max_tasks=max(n_tasks, 8), max_ctx=1024,
                      n_pages=max(64, 4 * n_tasks))
    eng = rt.Engine(None, p, v, flags=rt.RT_FLAG_TRACE if trace else rt.RT_FLAG_TIMING)
    for i in range(n_tasks):
        eng.submit(i % 64, [1, 2, 3], 0, 1_000_000, -2.0, 1.0, 90000, script=[5] * 600)
    for _ in range(5):
        eng.step()
    eng.sync()
    eng.reset_stats()
    t0 = time.perf_counter()
    for _ in range(rounds):
        eng.step()
    eng.sync()
    host_us = (time.perf_counter() - t0) / rounds * 1e6
    if trace:   # in-kernel phase marks (tools/trace_step.py)
        import numpy as np
        import trace_step
        agg, _, _, ph = trace_step.analyse(eng.trace())
        eng.close()
        body = {k: v[3] / v[0] for k, v in agg.items()}
        pre = np.median(np.array(ph["sched_pre"]), axis=0)
        return body, pre
    st = eng.stats()
    eng.close()
    return st["sched_ms"] / max(st["rounds"], 1) * 1e3, host_us


def main():
    if "--trace" in sys.argv:
        for n in [1, 8, 256, 2048]:
            body, pre = run(n, rounds=50, trace=True)
            print(f"N={n:5d}: sched_pre body {body.get('sched_pre', 0):6.1f} us, sched_post "
                  f"{body.get('sched_post', 0):6.1f} us; sched_pre phases (us) ingest | score | sort | "
                  "wcet+cand | admit | assemble | page pops | rows + publish: "
                  + " ".join(f"{x:.2f}" for x in pre), flush=True)
        return
    res = []
    for n in [1, 2, 4, 6, 8, 64, 256, 1024, 2048]:
        dev_us, host_us = run(n)
        res.append(dict(n_tasks=n, device_us_per_round=dev_us, host_us_per_round=host_us))
        print(f"N={n:5d}: device sched {dev_us:7.1f} us/round   rt_step wall {host_us:7.1f} us", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
