"""Pins for the comparison systems on the same engine (PAPER.md:576-584 the
baselines "vLLM" and "vLLM-stream", PAPER.md:657-661 the Seg-FCFS / Seg-EDF ablations):
segmentation modes SUSPEND (the method) / STREAM / NONE and the WCET-gate switch.

What the paper fixes and these pin:
* the plan "mu(100);mf(60)" is delivered as two executable segments + EOS by
  the method and by vLLM-stream (same boundaries: the stop checker is the same), but as ONE
  response at EOS by vLLM (no segmentation);
* vLLM-stream never suspends a generation (admitted once, decodes every round until EOS),
  while the method re-queues it after every segment;
* with a single request there is no contention, so the method's suspend / resume costs no
  round: its segment dispatch times equal vLLM-stream's exactly;
* vLLM's response time is the whole generation: W(s_0) = dispatch(EOS) + net - arrival;
* token fidelity (the concatenated segments are the response) in every mode, and the
  realized action durations do not depend on where boundaries fall (AMB-18 as re-read for
  NEXT-3), so completion time = response + sum of realized durations in vLLM.
"""
import pytest

from oracle.engine import (OracleEngine, STOP_EOS, STOP_SKILL, STOP_CAP, SEG_SUSPEND, SEG_STREAM, SEG_NONE,
                           SEG_MAX_TOKENS, FINISHED)
from oracle import agents
from synth import engine_params, compose_workload
from synth.configs import POLICY_FCFS, POLICY_EDF


def mk(vocab, **kw):
    p = engine_params("paper-4090", **kw)
    return OracleEngine(p, vocab.tok_skill, vocab.tok_exec_min_us, vocab.eos_id, vocab.vocab)


def tok(vocab, name):
    return [t for t, n in vocab.names.items() if n == name][0]


def run_one(v, mode, plan, window=0):
    e = mk(v, max_ctx=64, n_pages=8, seg_mode=mode, wcet_off=int(mode != SEG_SUSPEND))
    e.submit(0, [1, 2, 3], 0, 1_000_000, -2.0, 1.0, window, 0, script=plan)
    e.run_until_idle()
    return e, e.poll()


def test_plan_mu100_mf60_per_mode(tiny_vocab):
    v = tiny_vocab
    mu, mf, f = tok(v, "mu(100)"), tok(v, "mf(60)"), 3
    plan = [f, mu, f, mf, v.eos_id]
    got = {}
    for mode in (SEG_SUSPEND, SEG_STREAM, SEG_NONE):
        e, segs = run_one(v, mode, plan)
        got[mode] = segs
        assert sum((s["tokens"] for s in segs), []) == plan           # token fidelity
        assert [s["k"] for s in segs] == list(range(len(segs)))
        admitted = sum(len(r["admitted"]) for r in e.round_log)
        if mode == SEG_SUSPEND:
            assert admitted == 3                                      # re-queued per segment
        else:
            assert admitted == 1                                      # never suspended
    bounds = lambda segs: [(s["tok_begin"], s["tok_end"], s["reason"], s["n_skills"]) for s in segs]  # noqa: E731
    assert bounds(got[SEG_SUSPEND]) == [(0, 2, STOP_SKILL, 1), (2, 4, STOP_SKILL, 1), (4, 5, STOP_EOS, 0)]
    assert bounds(got[SEG_STREAM]) == bounds(got[SEG_SUSPEND])
    assert bounds(got[SEG_NONE]) == [(0, 5, STOP_EOS, 2)]
    assert got[SEG_NONE][0]["est_exec_us"] == v.tok_exec_min_us[mu] + v.tok_exec_min_us[mf]
    # no contention: suspend / resume costs no round -> identical dispatch times
    assert [s["dispatch_us"] for s in got[SEG_SUSPEND]] == [s["dispatch_us"] for s in got[SEG_STREAM]]
    assert got[SEG_NONE][0]["dispatch_us"] == got[SEG_STREAM][-1]["dispatch_us"]


def test_vllm_response_is_whole_generation(tiny_vocab):
    v = tiny_vocab
    mu, mf = tok(v, "mu(100)"), tok(v, "mf(60)")
    plan = [mu, 5, mf, 6, mu, v.eos_id]
    e, segs = run_one(v, SEG_NONE, plan)
    req = dict(request_id=segs[0]["request_id"], arrival_us=0, beta=1.0, alpha=-2.0, ert_us=1_000_000)
    m = agents.request_metrics(segs, req, v, e.p.net_us, seed=0)
    assert m["response_us"] == segs[0]["dispatch_us"] + e.p.net_us
    assert m["completion_us"] == m["response_us"] + m["exec_us"]
    # the same actions (segmentation-invariant realized durations) in the method's timeline
    e2, segs2 = run_one(v, SEG_SUSPEND, plan)
    m2 = agents.request_metrics(segs2, dict(req, request_id=segs2[0]["request_id"]), v, e2.p.net_us, seed=0)
    assert m2["exec_us"] == m["exec_us"]
    assert m2["response_us"] < m["response_us"]                        # first action earlier
    assert m2["completion_us"] <= m["completion_us"]                   # generation hidden behind actions


def test_stream_and_none_cut_at_max_tokens(tiny_vocab):
    v = tiny_vocab
    plan = [5] * (SEG_MAX_TOKENS + 7) + [v.eos_id]
    for mode in (SEG_STREAM, SEG_NONE):
        e = mk(v, max_ctx=256, n_pages=32, seg_mode=mode)
        e.submit(0, [1, 2], 0, 1_000_000, -2.0, 1.0, 0, 0, script=plan)
        e.run_until_idle()
        segs = e.poll()
        assert [(s["tok_end"] - s["tok_begin"], s["reason"]) for s in segs] == [(SEG_MAX_TOKENS, STOP_CAP),
                                                                                (8, STOP_EOS)]
        assert sum(len(r["admitted"]) for r in e.round_log) == 1


@pytest.mark.parametrize("mode,policy", [(SEG_NONE, POLICY_FCFS), (SEG_STREAM, POLICY_FCFS),
                                         (SEG_SUSPEND, POLICY_FCFS), (SEG_SUSPEND, POLICY_EDF)])
def test_modes_complete_and_keep_invariants(tiny_vocab, mode, policy):
    """Contended trace: every request completes, token fidelity per request, the free stack is
    whole at the end, and only the method re-queues generations."""
    v = tiny_vocab
    p = engine_params("paper-4090", max_batch=4, max_tasks=256, max_ctx=256, n_pages=48, policy=policy,
                      seg_mode=mode, wcet_off=int(mode != SEG_SUSPEND))
    reqs = compose_workload(16, 4.0, 8, range(1, 12), 8.0, 3, v, prompt_len_range=(10, 60), max_requests=80)
    e = OracleEngine(p, v.tok_skill, v.tok_exec_min_us, v.eos_id, v.vocab)
    for r in reqs:
        e.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, len(r.plan),
                 script=r.plan)
    e.run_until_idle()
    segs = e.poll()
    by = {}
    for s in segs:
        by.setdefault(s["request_id"], []).append(s)
    assert all(r.state == FINISHED for r in e.reqs.values())
    for rid, ss in by.items():
        assert sum((s["tokens"] for s in sorted(ss, key=lambda s: s["k"])), []) == e.reqs[rid].script
    assert len(e.free) == p.n_pages
    readmits = sum(len(r["admitted"]) for r in e.round_log) - len(e.reqs)
    assert (readmits > 0) == (mode == SEG_SUSPEND)
