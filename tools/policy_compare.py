"""Time utility of the method vs the paper's comparison systems on the same engine
(PAPER.md:576-584 baselines, 657-661 ablations, fig:diff-wl).

Every system runs the SAME synthetic trace through the device scheduler (scheduling-only
engine: scripted drone / robot-arm plans, no forward pass) with the VIRTUAL round clock of
the paper's hardware ("paper-4090": 21.77 ms per decoding iteration + batching, 114 us per
prefill token, SURVEY AMB-24), so the queueing the paper measured is reproduced:

  vLLM         FCFS, no segmentation (whole response at EOS), no WCET gate
  vLLM-stream  FCFS, segments streamed at skill boundaries, generation never suspended
  Seg-FCFS     segmentation + suspend/resume (the method's mechanism), FCFS order
  Seg-EDF      same, earliest initial deadline first
  Ours (PUD)   segmentation + Eq. 4 priority + WCET gate  (the method)

Workloads follow tab:data_sample: WID1 25 agents / 0.25 EPS / TPE 8 /
260 s, WID2 42 / 0.25 / 16 / 300 s, WID3 40 / 0.1 / 8 / 900 s (traces 1-8, drone prompts
1300 tokens) and ARM (robot-arm traces 9-11, prompt 2884).  Metrics:
mean time utility TUF_0(W(s_0)) per class, response time W(s_0), robot waiting time
sum_k W(s_k); realized action durations sampled identically for every system.

--oracle replays one workload through the CPU oracle and checks that the device produced
identical segment records (parity of the comparison itself).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import make_vocab, engine_params, compose_workload  # noqa: E402
from synth.configs import POLICY_PUD, POLICY_FCFS, POLICY_EDF, SEG_SUSPEND, SEG_STREAM, SEG_NONE  # noqa: E402
from synth.traces import TRACE_CLASSES  # noqa: E402
from paper_2412_18695_b200 import metrics  # noqa: E402

SYSTEMS = {
    "vLLM": dict(policy=POLICY_FCFS, seg_mode=SEG_NONE, wcet_off=1),
    "vLLM-stream": dict(policy=POLICY_FCFS, seg_mode=SEG_STREAM, wcet_off=1),
    "Seg-FCFS": dict(policy=POLICY_FCFS, seg_mode=SEG_SUSPEND, wcet_off=0),
    "Seg-EDF": dict(policy=POLICY_EDF, seg_mode=SEG_SUSPEND, wcet_off=0),
    "Ours (PUD)": dict(policy=POLICY_PUD, seg_mode=SEG_SUSPEND, wcet_off=0),
}
# chatbot (fig:chatbot): story generation read at 300 wpm; segments end at
# paragraphs (Ours-Para) or sentences (Ours-Sen) instead of skills; TUF of normal robot tasks
CHAT_SYSTEMS = {
    "vLLM": dict(policy=POLICY_FCFS, seg_mode=SEG_NONE, wcet_off=1, stop_grammar=2),
    "Ours-Para": dict(policy=POLICY_PUD, seg_mode=SEG_SUSPEND, wcet_off=0, stop_grammar=3, max_seg_tokens=16),
    "Ours-Sen": dict(policy=POLICY_PUD, seg_mode=SEG_SUSPEND, wcet_off=0, stop_grammar=2, max_seg_tokens=16),
}
WORKLOADS = {  # agents, EPS, max TPE, duration s, trace pool, prompt length
    "WID1": (25, 0.25, 8, 260.0, range(1, 9), 1300),
    "WID2": (42, 0.25, 16, 300.0, range(1, 9), 1300),
    "WID3": (40, 0.1, 8, 900.0, range(1, 9), 1300),
    "ARM": (16, 0.1, 4, 300.0, range(9, 12), 2884),
}


PREFIX = {1300: 1216, 2884: 2800}  # fixed prompt part pre-stored on the server (R-PFX)


def workload(name, vocab, seed, shared_prefix=True):
    """Requests + the shared fixed-prompt prefix (None without sharing).  Every system gets
    the same prefix: the fixed prompt components (skill set, guidance, examples) are stored
    server-side, so only the task part of a prompt is prefilled."""
    n, eps, tpe, dur, pool, pl = WORKLOADS[name]
    reqs = compose_workload(n, eps, tpe, pool, dur, seed, vocab, prompt_len_range=(pl, pl))
    if not shared_prefix:
        return reqs, None
    import numpy as np
    rng = np.random.Generator(np.random.PCG64([seed, 4242]))
    pre = rng.integers(0, vocab.vocab - 300, PREFIX[pl]).astype(np.int32)
    for r in reqs:
        r.prompt = np.concatenate([pre, np.asarray(r.prompt[len(pre):], dtype=np.int32)])
    return reqs, pre


def params(sysname, max_batch):
    return engine_params("paper-4090", max_batch=max_batch, max_tasks=2048, max_ctx=3072, n_pages=1 << 16,
                         **SYSTEMS[sysname])


def run_device(reqs, p, vocab, prefix=None):
    from paper_2412_18695_b200 import rt
    eng = rt.Engine(None, p, vocab)
    if prefix is not None:
        eng.register_prefix(prefix)
    rids = {}
    for r in reqs:
        rid = eng.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us,
                         len(r.plan), script=r.plan)
        rids[rid] = r
    segs = []
    rounds = 0
    done = set()
    while len(done) < len(reqs) and rounds < 2_000_000:
        eng.step()
        rounds += 1
        if rounds % 64 == 0:
            new = eng.poll()
            segs += new
            done |= {s["request_id"] for s in new if s["reason"] in (1, 2)}
    segs += eng.poll()
    eng.close()
    return segs, rids, rounds


def run_oracle(reqs, p, vocab, prefix=None):
    from oracle.engine import OracleEngine
    ora = OracleEngine(p, vocab.tok_skill, vocab.tok_exec_min_us, vocab.eos_id, vocab.vocab)
    if prefix is not None:
        ora.register_prefix(prefix)
    rids = {}
    for r in reqs:
        rids[ora.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us,
                        len(r.plan), script=r.plan)] = r
    ora.run_until_idle(max_rounds=2_000_000)
    return ora.poll(), rids


def summarize(segs, rids, vocab, net_us):
    reqd = {rid: dict(arrival_us=r.arrival_us, beta=r.beta, alpha=r.alpha, ert_us=r.ert_us,
                      cls=TRACE_CLASSES[r.trace_id]) for rid, r in rids.items()}
    rep = metrics.report(segs, reqd, vocab, net_us=net_us)
    return rep


def chat_workload(gv, seed, n=120, eps=0.5, dur=240.0):
    """Chat requests: Poisson arrivals, 64-token prompts, 2-3 paragraphs of 2-4 sentences."""
    import numpy as np
    from synth.grammar import chat_text
    rng = np.random.Generator(np.random.PCG64([seed, 77]))
    t, out = 0.0, []
    while len(out) < n:
        t += rng.exponential(1.0 / eps)
        if t >= dur:
            break
        out.append(dict(arrival_us=int(t * 1e6), prompt=rng.integers(0, gv.words[1], 64).astype(np.int32),
                        plan=chat_text(gv, rng, n_par=int(rng.integers(2, 4)))))
    return out


def run_chat(seed, max_batch, oracle=False):
    from synth.grammar import make_grammar_vocab
    gv = make_grammar_vocab(128256)
    reqs = chat_workload(gv, seed)
    res = {}
    for name, kw in CHAT_SYSTEMS.items():
        p = engine_params("paper-4090", max_batch=max_batch, max_tasks=2048, max_ctx=1024, n_pages=1 << 14, **kw)
        if oracle:
            from oracle.engine import OracleEngine
            eng = OracleEngine(p, gv.tok_skill, gv.tok_exec_min_us, gv.eos_id, gv.vocab, grammar=gv)
        else:
            from paper_2412_18695_b200 import rt
            eng = rt.Engine(None, p, gv)
        rids = {}
        for i, r in enumerate(reqs):
            rid = eng.submit(i % 64, r["prompt"], r["arrival_us"], 1_000_000, -2.0, 1.0, 0, len(r["plan"]),
                             script=r["plan"])
            rids[rid] = dict(arrival_us=r["arrival_us"], beta=1.0, alpha=-2.0, ert_us=1_000_000, cls="chat")
        segs = []
        if oracle:
            eng.run_until_idle(max_rounds=2_000_000)
            segs = eng.poll()
        else:
            done = set()
            for k in range(2_000_000):
                eng.step()
                if k % 64 == 63:
                    new = eng.poll()
                    segs += new
                    done |= {s["request_id"] for s in new if s["reason"] in (1, 2)}
                    if len(done) == len(reqs):
                        break
            segs += eng.poll()
            eng.close()
        rep = metrics.report(segs, rids, gv, net_us=p.net_us, exec_from="est")
        res[name] = {k: rep[k] for k in ("mean_utility", "mean_response_s", "mean_waiting_s", "n")}
    return dict(n_requests=len(reqs), systems=res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="WID1,WID2,WID3,ARM")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-batch", type=int, default=64)
    ap.add_argument("--oracle", action="store_true", help="also replay WID1 through the CPU oracle (parity)")
    ap.add_argument("--json", default=None)
    ap.add_argument("--no-prefix", action="store_true", help="prefill every prompt in full")
    ap.add_argument("--oracle-only", action="store_true", help="CPU oracle only (no GPU)")
    ap.add_argument("--chat", action="store_true", help="also the chatbot comparison (NEXT-4 grammars)")
    a = ap.parse_args()
    vocab = make_vocab(128256)
    out = dict(clock="paper-4090 VIRTUAL (PAPER.md:76, SURVEY AMB-24)", max_batch=a.max_batch,
               shared_prefix=not a.no_prefix, engine="oracle (CPU)" if a.oracle_only else "device scheduler",
               workloads={})
    for wname in a.workloads.split(","):
        reqs, pre = workload(wname, vocab, a.seed, shared_prefix=not a.no_prefix)
        res = {}
        for sname in SYSTEMS:
            p = params(sname, a.max_batch)
            t0 = time.perf_counter()
            if a.oracle_only:
                segs, rids = run_oracle(reqs, p, vocab, pre)
                rounds = -1
            else:
                segs, rids, rounds = run_device(reqs, p, vocab, pre)
            wall = time.perf_counter() - t0
            rep = summarize(segs, rids, vocab, p.net_us)
            rep["rounds"], rep["wall_s"] = rounds, wall
            res[sname] = rep
            if a.oracle and wname == a.workloads.split(",")[0]:
                osegs, orids = run_oracle(reqs, p, vocab, pre)
                key = lambda s: (s["request_id"], s["k"])  # noqa: E731
                same = sorted(segs, key=key) == sorted(osegs, key=key)
                rep["oracle_identical_segments"] = bool(same)
        base = res["vLLM"]
        ours = res["Ours (PUD)"]
        out["workloads"][wname] = dict(
            n_requests=len(reqs), systems=res,
            utility_ratio_vs_vllm=(ours["mean_utility"] / base["mean_utility"]
                                   if base["mean_utility"] > 0 else None),
            waiting_reduction_vs_vllm=1.0 - ours["mean_waiting_s"] / base["mean_waiting_s"])
        print(f"== {wname}: {len(reqs)} requests (paper-4090 virtual clock, batch {a.max_batch})")
        print(f"  {'system':12s} {'utility':>8s} {'response s':>10s} {'waiting s':>10s} {'rounds':>7s}  per class utility")
        for sname, rep in res.items():
            pc = " ".join(f"{c}={v['utility']:.3f}" for c, v in sorted(rep["by_class"].items()))
            print(f"  {sname:12s} {rep['mean_utility']:8.3f} {rep['mean_response_s']:10.3f} "
                  f"{rep['mean_waiting_s']:10.3f} {rep['rounds']:7d}  {pc}"
                  + (f"  oracle-identical={rep['oracle_identical_segments']}" if "oracle_identical_segments" in rep
                     else ""))
        w = out["workloads"][wname]
        r = w["utility_ratio_vs_vllm"]
        print(f"  PUD vs vLLM: utility x{r:.2f}" if r is not None else "  PUD vs vLLM: utility ratio n/a",
              f", waiting -{100 * w['waiting_reduction_vs_vllm']:.0f}%")
    if a.chat:
        out["chat"] = run_chat(a.seed, a.max_batch, oracle=a.oracle_only)
        print(f"== CHAT (story generation, 300 wpm reading): {out['chat']['n_requests']} requests")
        for sname, rep in out["chat"]["systems"].items():
            print(f"  {sname:12s} {rep['mean_utility']:8.3f} {rep['mean_response_s']:10.3f} {rep['mean_waiting_s']:10.3f}")
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
