"""Pins of the agent timeline and metrics (oracle c5 / c10), and parity of the product's
time-utility report (paper_2412_18695_b200/metrics.py) with the oracle.

Hand-worked examples (each value computed by hand from the definitions, not by the code
under test):
  * SPEC.md:394 ("8ms network latency"): an idle agent starts its action at
    dispatch + 8 ms;
  * SPEC.md:395 (fig:llm_time PAPER.md:281): a segment generated before the previous action
    ends waits 0 (W(s_k) = max(0, start_k - end_{k-1}));
  * SPEC.md:396 (fig:con_infer PAPER.md:217, "paralleled with the execution of the previous
    segment"): a segment dispatched during the previous action starts exactly at its end —
    the network latency is hidden;
  * one segment, arrival 0, action 0.5 s .. 2.5 s -> response 0.5, waiting 0.5,
    completion 2.5;
  * two back-to-back segments -> waiting = response;
  * SPEC.md:437 (PAPER.md:604 normal cut-off 1.5 s): response 1.5 s under the normal TUF ->
    utility 0.0.
"""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import agents
from oracle.engine import OracleEngine, SEG_SUSPEND, SEG_STREAM, SEG_NONE
from paper_2412_18695_b200 import metrics as M
from synth import engine_params, compose_workload, TRACE_CLASSES

NET = 8000


def fake_vocab(durations):
    """tokens 0..n-1 are skills with one realized duration each (µs); token n is filler."""
    n = len(durations)
    tok_skill = np.full(n + 1, -1, dtype=np.int16)
    tok_skill[:n] = 0
    return SimpleNamespace(tok_skill=tok_skill, realized={i: (d,) for i, d in enumerate(durations)})


def seg(k, dispatch_us, tokens, rid=7):
    return dict(request_id=rid, agent_id=0, k=k, tokens=list(tokens), dispatch_us=dispatch_us, reason=3,
                est_exec_us=0)


def test_idle_agent_starts_at_dispatch_plus_network():
    v = fake_vocab([1_000_000])
    tl = agents.simulate_request([seg(0, 300_000, [0])], 0, v, NET, 0, 7)
    assert tl[0]["start"] == 308_000 and tl[0]["end"] == 1_308_000 and tl[0]["W"] == 308_000


def test_segment_generated_during_previous_action_waits_zero():
    v = fake_vocab([2_000_000, 500_000])
    # segment 0 dispatched at 0.1 s -> action 0.108 .. 2.108 s; segment 1 dispatched at 0.2 s,
    # i.e. during action 0 (0.2 + 0.008 < 2.108): it starts at 2.108 s, the network hidden
    tl = agents.simulate_request([seg(0, 100_000, [0]), seg(1, 200_000, [1])], 0, v, NET, 0, 7)
    assert [x["start"] for x in tl] == [108_000, 2_108_000]
    assert [x["W"] for x in tl] == [108_000, 0]
    assert tl[1]["end"] == 2_608_000
    # dispatched after action 0 ended: the network latency is paid again (3.0 + 0.008 - 2.108)
    tl = agents.simulate_request([seg(0, 100_000, [0]), seg(1, 3_000_000, [1])], 0, v, NET, 0, 7)
    assert [x["W"] for x in tl] == [108_000, 900_000]


def test_spec_435_single_segment_metrics():
    v = fake_vocab([2_000_000])
    req = dict(request_id=7, arrival_us=0, beta=1.0, alpha=-2.0, ert_us=1_000_000)
    m = agents.request_metrics([seg(0, 492_000, [0])], req, v, NET, 0)
    assert (m["response_us"], m["waiting_us"], m["completion_us"]) == (500_000, 500_000, 2_500_000)
    assert m["utility"] == 1.0                                     # 0.5 s < ERT 1 s: utility beta


def test_spec_436_back_to_back_waiting_equals_response():
    v = fake_vocab([1_000_000, 1_000_000])
    req = dict(request_id=7, arrival_us=0, beta=1.0, alpha=-2.0, ert_us=1_000_000)
    m = agents.request_metrics([seg(0, 92_000, [0, 2]), seg(1, 600_000, [1])], req, v, NET, 0)
    assert m["response_us"] == 100_000 and m["waiting_us"] == 100_000
    assert m["completion_us"] == 2_100_000


def test_spec_437_normal_tuf_response_1_5s_utility_zero():
    v = fake_vocab([1_000_000])
    req = dict(request_id=7, arrival_us=0, beta=1.0, alpha=-2.0, ert_us=1_000_000)
    m = agents.request_metrics([seg(0, 1_492_000, [0])], req, v, NET, 0)
    assert m["response_us"] == 1_500_000 and m["utility"] == 0.0
    # the urgent preset (beta 2, alpha -6.67, ERT 0.2 s) at its 0.5 s cut-off: 2 - 6.67 * 0.3
    req_u = dict(req, beta=2.0, alpha=-6.67, ert_us=200_000)
    m = agents.request_metrics([seg(0, 492_000, [0])], req_u, v, NET, 0)
    assert m["utility"] == pytest.approx(-0.001, abs=1e-12)


@pytest.mark.parametrize("mode", [SEG_SUSPEND, SEG_STREAM, SEG_NONE])
def test_product_report_equals_oracle_metrics(tiny_vocab, mode):
    """metrics.report (the bench's time_utility / time_utility_systems) against the oracle's
    request_metrics + aggregate on the same segment logs, per request and per class, for every
    serving mode (rt.h RT_SEG_*)."""
    v = tiny_vocab
    p = engine_params("paper-4090", max_batch=4, max_tasks=256, max_ctx=256, n_pages=64, seg_mode=mode,
                      wcet_off=int(mode != SEG_SUSPEND))
    reqs = compose_workload(12, 3.0, 6, range(1, 12), 10.0, 5, v, prompt_len_range=(10, 60), max_requests=60)
    e = OracleEngine(p, v.tok_skill, v.tok_exec_min_us, v.eos_id, v.vocab)
    info = {}
    for r in reqs:
        rid = e.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, len(r.plan),
                       script=r.plan)
        info[rid] = dict(request_id=rid, arrival_us=r.arrival_us, beta=r.beta, alpha=r.alpha, ert_us=r.ert_us,
                         cls=TRACE_CLASSES[r.trace_id])
    e.run_until_idle()
    segs = e.poll()
    for seed in (0, 11):
        got = M.report(segs, info, v, net_us=p.net_us, seed=seed, per_request=True)
        by = {}
        for s in segs:
            by.setdefault(s["request_id"], []).append(s)
        ora = [agents.request_metrics(by[rid], info[rid], v, p.net_us, seed) for rid in sorted(by)]
        assert len(got["requests"]) == len(ora) == len(reqs)
        for g, o in zip(sorted(got["requests"], key=lambda m: m["request_id"]), ora):
            for key in ("response_us", "waiting_us", "completion_us", "exec_us", "utility"):
                assert g[key] == o[key], (key, g, o)
        agg = agents.aggregate(ora)
        assert set(got["by_class"]) == set(agg)
        for c, a in agg.items():
            for key in ("n", "utility", "response_s", "waiting_s"):
                assert got["by_class"][c][key] == pytest.approx(a[key], rel=1e-12, abs=1e-12), (c, key)
