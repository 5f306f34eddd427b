"""Where the e2e closed loop spends its rounds (bench.py `e2e`, shared drone prefix): per
round the forward rows (decode + prompt), the device step time (CUDA events, RT_FLAG_TIMING)
and the host wall time of the rt_step call; aggregated by rows bucket."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import bench  # noqa: E402
import profile_step  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402
from synth.traces import system_prefix  # noqa: E402


def main(rounds=200, trace=False):
    wl = os.environ.get("WORKLOAD", "C3")
    eng, now = profile_step.setup(None, flags=rt.RT_FLAG_TRACE if trace else rt.RT_FLAG_TIMING, workload=wl)
    from synth import MODEL_SHAPES, make_vocab
    from paper_2412_18695_b200 import replicas as R
    vocab = make_vocab(MODEL_SHAPES["llama3-8b"].vocab)
    R.lockstep_until_idle(lambda: eng.step(now()), None, max_rounds=4000)
    eng.poll()
    pfx = {r: system_prefix(vocab, r, bench.PREFIX[r], seed=0) for r in ("drone", "arm")}
    for r in ("drone", "arm"):
        eng.register_prefix(pfx[r])
    ordinal = {}

    pregen = {}   # as bench.py: request generation is the harness's work, outside the loop

    def submit(agent):
        o = ordinal[agent] = ordinal.get(agent, 0) + 1
        tr = pregen.pop((agent, o), None) or bench.agent_request(wl, vocab, agent, o, 0, prefixes=pfx)
        eng.submit(agent, tr.prompt, now(), tr.ert_us, tr.alpha, tr.beta, 90000, script=tr.plan)

    for a in range(bench.WORKLOADS[wl]["agents"]):
        for o in range(2, 8):
            pregen[(a, o)] = bench.agent_request(wl, vocab, a, o, 0, prefixes=pfx)
        submit(a)
    if trace:   # closed loop for a while, then the device trace of 10 rounds by kernel role
        for r in range(60):
            for s in eng.poll():
                if s["reason"] in (1, 2):
                    submit(s["agent_id"])
            eng.step(now())
        eng.sync()
        eng.reset_stats()
        # E2E_PIPELINED=1: step, then drain the retired rounds (rt_poll_segment_ready) and
        # resubmit while the round runs — no host gap, but every resubmission is admitted one
        # round later (measured in bench's closed loop: 9.7 k vs 10.1 k tok/s, not adopted)
        pipelined = os.environ.get("E2E_PIPELINED", "0") == "1"
        for r in range(10):
            if pipelined:   # bench.py's e2e loop: step, then the retired rounds' segments
                eng.step(now())
                for s in eng.poll(wait=False):
                    if s["reason"] in (1, 2):
                        submit(s["agent_id"])
            else:
                for s in eng.poll():
                    if s["reason"] in (1, 2):
                        submit(s["agent_id"])
                eng.step(now())
        eng.sync()
        import trace_step
        agg, span, n, ph = trace_step.analyse(eng.trace())
        print(f"e2e trace: {n} launches, {span / 10:.0f} us per round (gap = from the previous launch's "
              "exit to this launch's dependency release: for sched_pre it holds the host's poll / submit)")
        for name, (cnt, lead, gap, body, ctas, mains, epis) in sorted(agg.items(), key=lambda x: -(x[1][2] + x[1][3])):
            print(f"  {name:28s} n={cnt:5d} per round: gap {gap / 10:9.1f} us, body {body / 10:9.1f} us "
                  f"(body per launch {body / cnt:8.1f} us)")
        for name, v in ph.items():
            if name.startswith("sched"):
                print(f"{name} phases (median us): ingest | score | sort | wcet+candidates | admit | assemble | "
                      "page pops | rows + publish")
                print("  " + " ".join(f"{x:7.2f}" for x in np.median(np.array(v), axis=0)))
        eng.close()
        return
    rec = []
    for r in range(rounds):
        for s in eng.poll():
            if s["reason"] in (1, 2):
                submit(s["agent_id"])
        eng.sync()
        t0 = time.perf_counter()
        info = eng.step(now())
        eng.sync()
        wall = (time.perf_counter() - t0) * 1e3
        st = eng.stats()   # cumulative; this round's CUDA-event timing was harvested by rt_sync
        rec.append([info["n_rows"], info["n_prefill_rows"], info["n_running"], wall,
                    st["step_ms"], st["gemm_ms"], st["attn_ms"]])
    a = np.array(rec, dtype=np.float64)
    a[1:, 4:7] = a[1:, 4:7] - a[:-1, 4:7]   # round r's device times = stats after r - after r-1
    a = a[20:]
    print(f"rounds {len(a)}: mean rows {a[:, 0].mean():.0f} (prompt {a[:, 1].mean():.0f}), tokens/round "
          f"{a[:, 2].mean():.1f}, wall {a[:, 3].mean():.2f} ms, device {a[:, 4].mean():.2f} ms "
          f"(forward {a[:, 5].mean():.2f}, attention {a[:, 6].mean():.2f}) -> {a[:, 2].sum() / a[:, 3].sum() * 1e3:.0f} tok/s")
    big = a[a[:, 0] >= 513, 0]
    if len(big):
        print("  rows of the > 512-row rounds: percentiles 10/50/90 =", np.percentile(big, [10, 50, 90]).round())
    for lo, hi in ((0, 65), (65, 129), (129, 257), (257, 513), (513, 100000)):
        m = (a[:, 0] >= lo) & (a[:, 0] < hi)
        if m.any():
            b = a[m]
            print(f"  rows [{lo:4d},{hi:6d}): {m.sum():4d} rounds, wall {b[:, 3].mean():6.2f} ms, device "
                  f"{b[:, 4].mean():6.2f} ms, forward {b[:, 5].mean():6.2f} ms, attention {b[:, 6].mean():5.2f} ms")
    eng.close()


if __name__ == "__main__":
    main(trace=len(sys.argv) > 1 and sys.argv[1] == "trace")
