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
from synth import make_vocab, engine_params  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def run(n_tasks, rounds=200):
    v = make_vocab(512)
    p = engine_params("b200-roofline", max_batch=1, max_tasks=max(n_tasks, 8), max_ctx=1024,
                      n_pages=max(64, 4 * n_tasks))
    eng = rt.Engine(None, p, v, flags=rt.RT_FLAG_TIMING)
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
    st = eng.stats()
    eng.close()
    return st["sched_ms"] / max(st["rounds"], 1) * 1e3, host_us


def main():
    res = []
    for n in [1, 2, 4, 6, 8, 64, 256, 1024, 2048]:
        dev_us, host_us = run(n)
        res.append(dict(n_tasks=n, device_us_per_round=dev_us, host_us_per_round=host_us))
        print(f"N={n:5d}: device sched {dev_us:7.1f} us/round   rt_step wall {host_us:7.1f} us", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
