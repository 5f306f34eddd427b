"""Pins for the oracle round loop: WCET gate (P4), stop checker (P5), allocator
invariants (P8), metrics identities (P10), determinism (P11), FCFS degenerate
case (c11), a hand-worked urgent-vs-normal trace, deadlock freedom (R-MEM)."""
import math

import numpy as np
import pytest

from oracle.engine import (OracleEngine, wcet_gate_pass, STOP_EOS, STOP_SKILL, STOP_CAP,
                           STOP_MAXNEW, FINISHED, OracleError, ceil_div)
from oracle import agents
from synth import engine_params, compose_workload
from synth.configs import POLICY_FCFS


def mk(vocab, **kw):
    p = engine_params("paper-4090", **kw)
    return OracleEngine(p, vocab.tok_skill, vocab.tok_exec_min_us, vocab.eos_id, vocab.vocab)


def tok(vocab, name):
    return [t for t, n in vocab.names.items() if n == name][0]


def test_p4_wcet_gate():
    # 3 of 10 tokens done, 21.77 ms/token (tab:latency PAPER.md:76)
    hist = [21770] * 5
    assert wcet_gate_pass(10, 3, sum(hist), 5, 200000)          # 152.39 ms <= 200 ms
    assert not wcet_gate_pass(10, 3, sum(hist), 5, 100000)      # 152.39 ms  > 100 ms
    assert wcet_gate_pass(10, 3, 0, 0, -1)                      # no speed history -> admit
    assert 7 * 21770 == 152390


def test_p5_stop_checker_plan_mu100_mf50(tiny_vocab):
    v = tiny_vocab
    mu, mf = tok(v, "mu(100)"), tok(v, "mf(60)")
    f = 3  # filler (non-skill)
    plan = [f, mu, f, mf, v.eos_id]        # "mu(100);mf(60)" then EOS
    for window, expect in [(0, [(2, STOP_SKILL), (2, STOP_SKILL), (1, STOP_EOS)]),
                           (10_000_000, [(5, STOP_EOS)])]:
        e = mk(v, max_ctx=64, n_pages=8)
        e.submit(0, [1, 2, 3], 0, 1_000_000, -2.0, 1.0, window, 0, script=plan)
        e.run_until_idle()
        segs = e.poll()
        assert [(s["tok_end"] - s["tok_begin"], s["reason"]) for s in segs] == expect
        assert sum((s["tokens"] for s in segs), []) == plan           # token fidelity
        if window == 0:
            assert [s["n_skills"] for s in segs] == [1, 1, 0]
            assert segs[0]["est_exec_us"] == v.tok_exec_min_us[mu]
        else:
            assert segs[0]["n_skills"] == 2
            assert segs[0]["est_exec_us"] == v.tok_exec_min_us[mu] + v.tok_exec_min_us[mf]


def test_p5_filler_and_cap(tiny_vocab):
    v = tiny_vocab
    plan = [5] * 25 + [v.eos_id]
    e = mk(v, max_ctx=64, n_pages=8)
    e.submit(0, [1, 2], 0, 1_000_000, -2.0, 1.0, 0, 0, script=plan)
    e.run_until_idle()
    segs = e.poll()
    assert [(s["tok_begin"], s["tok_end"], s["reason"]) for s in segs] == [
        (0, 10, STOP_CAP), (10, 20, STOP_CAP), (20, 26, STOP_EOS)]
    assert all(s["n_skills"] == 0 and s["est_exec_us"] == 0 for s in segs)
    # MAXNEW: a script without EOS ends the request at its last token
    e = mk(v, max_ctx=64, n_pages=8)
    e.submit(0, [1, 2], 0, 1_000_000, -2.0, 1.0, 0, 0, script=[5, 6, 7])
    e.run_until_idle()
    assert [s["reason"] for s in e.poll()] == [STOP_MAXNEW]


def test_window_reading_amb11(tiny_vocab):
    # window 90 ms with ~1 ms print skills merges several skills into one segment
    v = tiny_vocab
    p = tok(v, "p()")
    plan = [p, 4, p, 4, p, v.eos_id]
    e = mk(v, max_ctx=64, n_pages=8)
    e.submit(0, [1], 0, 1_000_000, -2.0, 1.0, 90000, 0, script=plan)
    e.run_until_idle()
    segs = e.poll()
    assert [(s["tok_end"] - s["tok_begin"], s["n_skills"]) for s in segs] == [(6, 3)]


def run_c1(v, seed=0, policy=None, check=None, **kw):
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, seed, v, prompt_len_range=(40, 64),
                            max_requests=12)
    extra = dict(max_ctx=256, n_pages=64, max_batch=4, max_tasks=64)
    extra.update(kw)
    if policy is not None:
        extra["policy"] = policy
    e = mk(v, **extra)
    ids = {}
    for r in reqs:
        ids[e.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta,
                     r.exec_window_us, 0, script=r.plan)] = r
    for _ in range(10000):
        info = e.step()
        if check:
            check(e, info)
        if info["n_running"] == 0 and all(x.state == FINISHED for x in e.reqs.values()):
            break
    return e, ids


def test_p8_allocator_invariants(tiny_vocab):
    P = 16

    def check(e, info):
        held = sum(len(r.pages) for r in e.reqs.values())
        assert len(e.free) + held == e.p.n_pages
        for r in e.reqs.values():
            if r.holder:
                assert len(r.pages) == ceil_div(r.ctx, P)
        assert sum(r.R - len(r.pages) for r in e.reqs.values() if r.holder) <= len(e.free)
        all_pages = [pg for r in e.reqs.values() for pg in r.pages] + e.free
        assert sorted(all_pages) == list(range(e.p.n_pages))
    e, _ = run_c1(tiny_vocab, check=check)
    assert all(r.state == FINISHED for r in e.reqs.values())
    assert sorted(e.free) == list(range(64))


def test_p8_kv_size_matches_paper():
    from synth import MODEL_SHAPES
    s = MODEL_SHAPES["llama3-8b"]
    assert s.kv_bytes_per_token == 131072
    assert s.kv_bytes_per_token * 1300 / 1e6 == pytest.approx(170.35, abs=0.1)


def test_allocator_first_pops_are_0_1_2(tiny_vocab):
    v = tiny_vocab
    e = mk(v, max_ctx=128, n_pages=16)
    e.submit(0, list(range(1, 34)), 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5] * 20)   # 3 pages
    e.submit(1, list(range(1, 10)), 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5] * 20)   # 1 page
    e.step()
    tabs = e.page_tables()
    assert tabs[0] == [0, 1, 2] and tabs[1] == [3]
    e.step()   # decode: request 0 ctx 33 -> no pop ; request 1 ctx 9 -> no pop
    assert e.page_tables() == {0: [0, 1, 2], 1: [3]}


def test_p10_metrics_identities_and_p11_determinism(tiny_vocab):
    v = tiny_vocab
    e1, ids = run_c1(v, seed=3)
    e2, _ = run_c1(v, seed=3)
    s1, s2 = e1.poll(), e2.poll()
    assert s1 == s2
    assert [{k: x for k, x in r.items() if k != "logits"} for r in e1.round_log] == \
        [{k: x for k, x in r.items() if k != "logits"} for r in e2.round_log]
    ms = []
    for rid, r in ids.items():
        segs = [s for s in s1 if s["request_id"] == rid]
        m = agents.request_metrics(segs, dict(request_id=rid, arrival_us=r.arrival_us, beta=r.beta,
                                              alpha=r.alpha, ert_us=r.ert_us, cls=r.trace_id),
                                   v, 8000, 0)
        ms.append(m)
        assert m["completion_us"] == m["waiting_us"] + m["exec_us"]          # C = sum(W + E)
        assert m["response_us"] <= m["waiting_us"]
        assert m["utility"] <= r.beta
    agg = agents.aggregate(ms)
    assert sum(a["n"] for a in agg.values()) == 12


def test_fcfs_policy_dispatch_order(tiny_vocab):
    # c11: FCFS never reorders first dispatches; batch 1 serialises
    e, ids = run_c1(tiny_vocab, seed=1, policy=POLICY_FCFS, max_batch=1)
    segs = e.poll()
    first = [s["request_id"] for s in segs if s["k"] == 0]
    arr = sorted(ids, key=lambda rid: (ids[rid].arrival_us, rid))
    assert first == arr


def test_pud_reduces_to_fcfs_on_same_class_predeadline(tiny_vocab):
    v = tiny_vocab
    outs = []
    for pol in (0, POLICY_FCFS):
        e = mk(v, max_ctx=128, n_pages=64, max_batch=1, base_us=1000, gamma_ppm=0,
               prefill_us_per_tok=0, policy=pol)
        for i in range(5):
            e.submit(i, [1, 2, 3], 1000 * i, 10 ** 6, -2.0, 1.0, 0, 0, script=[5, 5, v.eos_id])
        e.run_until_idle()
        outs.append([(s["request_id"], s["k"]) for s in e.poll()])
    # all k=0 and pre-deadline: identical admission order
    assert [x for x in outs[0] if x[1] == 0] == [x for x in outs[1] if x[1] == 0]


def test_hand_worked_urgent_preempts_normal(tiny_vocab):
    """Task 71/72 story at batch 1 with the paper-4090 clock.

    Round 0 (t=0): only the normal request (arrived 0) is waiting -> admitted,
      prefill of 3 tokens: round_us = 21770 + 114*3 = 22112.
    Round 1 (t=22112): urgent arrived at 10000 is waiting; batch is full (1 slot)
      -> normal decodes, round_us = 21770.  Its 2nd token mu(..) completes a
      segment (window 0): suspend, D := dispatch + net + E_min.
    Round 2 (t=43882): both waiting; urgent Pri ~ 2/(0.09*0.0939)... >> normal
      (k=1, L ~ seconds) -> urgent admitted."""
    v = tiny_vocab
    mu = tok(v, "mu(100)")
    e = mk(v, max_ctx=64, n_pages=8, max_batch=1)
    n = e.submit(0, [1, 2, 3], 0, 1_000_000, -2.0, 1.0, 0, 0, script=[4, mu, 4, v.eos_id])
    u = e.submit(1, [1, 2, 3], 10000, 200000, -6.67, 2.0, 0, 0, script=[mu, v.eos_id])
    i0 = e.step()
    assert (i0["t_us"], i0["round_us"], e.round_log[-1]["admitted"]) == (0, 22112, [n])
    i1 = e.step()
    assert (i1["t_us"], i1["round_us"], i1["n_admitted"], i1["n_stopped"]) == (22112, 21770, 0, 1)
    seg = e.poll()[0]
    assert seg["dispatch_us"] == 22112 + 21770 and seg["reason"] == STOP_SKILL
    assert e.reqs[n].D == 43882 + 8000 + v.tok_exec_min_us[mu]
    e.step()
    assert e.round_log[-1]["admitted"] == [u]
    assert e.round_log[-1]["t_us"] == 43882


def test_memory_pressure_no_deadlock(tiny_vocab):
    # R-MEM reading: a k=0 head that does not fit must not block k>0 resumes
    v = tiny_vocab
    mu = tok(v, "mu(100)")
    e = mk(v, max_ctx=64, n_pages=6, max_batch=4)
    for i in range(4):
        e.submit(i, list(range(1, 20)), i, 1_000_000, -2.0, 1.0, 0, 0,
                 script=[mu, 4, mu, 4, mu, v.eos_id])     # R = ceil(25/16) = 2 pages each
    e.run_until_idle(max_rounds=2000)
    segs = e.poll()
    assert sum(1 for s in segs if s["reason"] == STOP_EOS) == 4
    assert sorted(e.free) == list(range(6))
    assert any(r["n_refused_mem"] > 0 for r in e.round_log)


def test_submit_validation(tiny_vocab):
    v = tiny_vocab
    e = mk(v, max_ctx=64, n_pages=2, max_tasks=2)
    with pytest.raises(OracleError) as ex:
        e.submit(0, [1], 0, 10 ** 6, 0.5, 1.0, 0, 0, script=[5])      # alpha > 0
    assert ex.value.code == "INVAL"
    with pytest.raises(OracleError):
        e.submit(0, [1], 0, -1, -1.0, 1.0, 0, 0, script=[5])          # ERT < 0
    with pytest.raises(OracleError):
        e.submit(0, [1], 0, 10, -1.0, math.inf, 0, 0, script=[5])     # beta not finite
    with pytest.raises(OracleError):
        e.submit(0, [512], 0, 10, -1.0, 1.0, 0, 0, script=[5])        # token id out of range
    with pytest.raises(OracleError):
        e.submit(0, [1] * 60, 0, 10, -1.0, 1.0, 0, 0, script=[5] * 10)  # > max_ctx
    with pytest.raises(OracleError) as ex:
        e.submit(0, [1] * 40, 0, 10, -1.0, 1.0, 0, 0, script=[5])     # 3 pages > pool of 2
    assert ex.value.code == "NOMEM"


def test_wcet_lag_for_one_generation_hand_worked(tiny_vocab):
    """Reading R-WCET ("By introducing a lag for one generation,
    this method offers a profiling-independent strategy"): the gate of round r uses the speed
    measured through round r-1 — no batch-latency model, unlike SPEC.md:325's scaled WCET.
    Hand-worked on the paper-4090 VIRTUAL clock (base 21770 us, gamma 5 %, prefill 114 us/token),
    max_admit_per_round = 1 (the paper's incremental growth), 1-token prompts, filler scripts:
      round 0  t = 0       A admitted alone (no history); latency 21770 + 114 = 21884
      round 1  t = 21884   gate protects A: D_A - t = 220000 - 21884 = 198116;
                           (10 - 1) * 21884 = 196956 <= 198116 -> B admitted
                           (SPEC's scaled rule: 196956 * 22858 / 21770 = 206799 > 198116 would refuse)
                           latency 21770 + floor(21770 * 0.05) + 114 = 22972
      round 2  t = 44856   D_A - t = 175144, n = 2, S = 44856: 8 * 44856 = 358848 > 2 * 175144 = 350288
                           -> C refused (the gate sees the grown latency one generation later)
    A's 10-token segment (CAP) then ends at 21884 + 22972 + 8 * 22858 = 227720: 7720 us past its
    deadline — the overrun the one-generation lag allows (bounded by the latency growth of the
    admissions the gate has not yet seen)."""
    v = tiny_vocab
    e = mk(v, max_batch=4, max_tasks=8, max_ctx=64, n_pages=16, max_admit_per_round=1)
    filler = [5] * 30 + [v.eos_id]
    ra = e.submit(0, [1], 0, 220_000, -2.0, 1.0, 0, 0, script=filler)
    rb = e.submit(1, [1], 1, 100_000_000, -2.0, 1.0, 0, 0, script=filler)
    rc = e.submit(2, [1], 2, 100_000_000, -2.0, 1.0, 0, 0, script=filler)
    i0 = e.step()
    assert (i0["t_us"], i0["n_admitted"], e.round_log[-1]["admitted"]) == (0, 1, [ra])
    i1 = e.step()
    assert (i1["t_us"], i1["n_admitted"], i1["n_refused_wcet"], e.round_log[-1]["admitted"]) == (21884, 1, 0, [rb])
    i2 = e.step()
    assert (i2["t_us"], i2["n_admitted"], i2["n_refused_wcet"]) == (44856, 0, 1)
    assert 9 * 21884 == 196956 and 196956 * 22858 // 21770 == 206799
    while True:
        e.step()
        segs = [s for s in e.poll() if s["request_id"] == ra]
        if segs:
            break
    assert segs[0]["reason"] == STOP_CAP and segs[0]["tok_end"] == 10
    assert segs[0]["dispatch_us"] == 21884 + 22972 + 8 * 22858 == 227720
