"""Pins for KV eviction to host memory + restore (PAPER.md:226-229 context
caching in host memory; reading R-EVICT).

* The paper's restore-vs-re-prefill trade is about a suspended generation's KV: 8B KV is
  131072 B per token, so a 1300-token drone context is 82 pages of 2 MiB
  = 170.4 MB (170.35 MB).
* Conservation every round: device free pages + pages held by holders (+ registered prefix
  pages) = pool; host free pages + host pages held by evicted requests = host pool; an
  evicted request holds no device page and is not a holder.
* A restore brings back exactly the host pages the request was evicted to (same count, same
  order); every request still finishes with its scripted tokens (no re-prefill, KV kept).
* The point of the mechanism: a high-priority request that does not fit is admitted at once
  by evicting lower-priority suspended contexts, instead of waiting for one to finish.
* All-or-nothing: no eviction when evicting every eligible victim would still not fit.
"""
from oracle.engine import OracleEngine, FINISHED, ceil_div
from synth import engine_params, compose_workload


def mk(vocab, **kw):
    p = engine_params("paper-4090", **kw)
    return OracleEngine(p, vocab.tok_skill, vocab.tok_exec_min_us, vocab.eos_id, vocab.vocab)


def tok(vocab, name):
    return [t for t, n in vocab.names.items() if n == name][0]


def check_conservation(e):
    p = e.p
    held = sum(len(r.pages) - r.npfx for r in e.reqs.values() if r.holder)
    pfx = sum(len(x["pages"]) for x in e.prefixes)
    assert len(e.free) + held + pfx == p.n_pages
    hheld = sum(len(r.hpages) for r in e.reqs.values() if r.evicted)
    assert len(e.hfree) + hheld == e.host_pages
    for r in e.reqs.values():
        if r.evicted:
            assert not r.holder and len(r.pages) == r.npfx and len(r.hpages) == ceil_div(r.ctx, p.page_tokens) - r.npfx
    assert e._avail() >= 0


def test_kv_bytes_per_page_matches_paper():
    per_tok = 32 * 2 * 8 * 128 * 2                    # 8B: layers x (K, V) x kv heads x hd x bf16
    assert per_tok == 131072
    pages = ceil_div(1300, 16)
    assert pages == 82
    assert abs(1300 * per_tok / 1e6 - 170.35) < 0.1


def urgent_scenario(v, host_pages):
    mu, mf, f = tok(v, "mu(100)"), tok(v, "mf(60)"), 3
    long_plan = [f, mu, f, mf, f, mu, f, mf, f, mu, f, mf] * 3 + [v.eos_id]     # many suspensions
    e = mk(v, max_batch=2, max_tasks=16, max_ctx=96, n_pages=12, host_pages=host_pages, swap_us_per_page=116)
    for a in range(2):      # two normal requests take 10 of 12 pages (R = ceil((40 + 37) / 16) = 5 each)
        e.submit(a, list(range(1, 41)), 0, 1_000_000, -2.0, 1.0, 0, 0, script=long_plan)
    urg = e.submit(9, list(range(50, 90)), 300_000, 200_000, -6.67, 2.0, 0, 0, script=[mu, v.eos_id])
    first = None
    for _ in range(400):
        info = e.step()
        check_conservation(e)
        if first is None:
            first = next((s for s in e.segments if s["request_id"] == urg), None)
        if info["n_running"] == 0 and all(r.state == FINISHED for r in e.reqs.values()):
            break
    segs = e.poll()
    return e, segs, first


def test_eviction_admits_urgent_request_early(tiny_vocab):
    v = tiny_vocab
    e0, s0, f0 = urgent_scenario(v, 0)
    e1, s1, f1 = urgent_scenario(v, 16)
    assert sum(r["n_evicted"] for r in e0.round_log) == 0
    assert sum(r["n_evicted"] for r in e1.round_log) >= 1
    assert sum(r["n_restored"] for r in e1.round_log) == sum(r["n_evicted"] for r in e1.round_log)
    assert f1["dispatch_us"] < f0["dispatch_us"]                      # admitted without waiting
    for e, segs in ((e0, s0), (e1, s1)):                              # fidelity, all finished
        by = {}
        for s in segs:
            by.setdefault(s["request_id"], []).extend(s["tokens"])
        assert all(by[rid] == r.script for rid, r in e.reqs.items())
    # restores bring back exactly the host pages of the eviction, in order
    ev, rs = {}, {}
    for r in e1.round_log:
        for d, rid, dp, hp in r["swaps"]:
            (ev if d == 0 else rs).setdefault(rid, []).append(hp)
    assert ev and set(ev) == set(rs)
    for rid in ev:
        assert rs[rid][:len(ev[rid])] == ev[rid][:len(rs[rid])]
    assert len(e1.free) == e1.p.n_pages and len(e1.hfree) == e1.host_pages


def test_no_eviction_when_it_cannot_fit(tiny_vocab):
    v = tiny_vocab
    mu, f = tok(v, "mu(100)"), 3
    e = mk(v, max_batch=4, max_tasks=16, max_ctx=200, n_pages=8, host_pages=16)
    e.submit(0, list(range(1, 41)), 0, 1_000_000, -2.0, 1.0, 0, 0, script=[f, mu, f, mu, v.eos_id])
    # needs ceil((120 + 2) / 16) = 8 pages: never fits while request 0 runs or holds 3+ pages
    big = e.submit(1, list(range(1, 121)), 100_000, 200_000, -6.67, 2.0, 0, 0, script=[mu, v.eos_id])
    for _ in range(200):
        e.step()
        check_conservation(e)
        if all(r.state == FINISHED for r in e.reqs.values()):
            break
    assert all(r.state == FINISHED for r in e.reqs.values())
    assert sum(r["n_evicted"] for r in e.round_log) in (0, 1)
    assert e.reqs[big].state == FINISHED


def test_eviction_under_contention_keeps_invariants(tiny_vocab):
    v = tiny_vocab
    p = engine_params("paper-4090", max_batch=8, max_tasks=512, max_ctx=256, n_pages=40, host_pages=64,
                      swap_us_per_page=116)
    reqs = compose_workload(24, 6.0, 8, range(1, 12), 8.0, 9, v, prompt_len_range=(20, 90), max_requests=120)
    e = OracleEngine(p, v.tok_skill, v.tok_exec_min_us, v.eos_id, v.vocab)
    for r in reqs:
        e.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, len(r.plan),
                 script=r.plan)
    for _ in range(100000):
        info = e.step()
        check_conservation(e)
        if info["n_running"] == 0 and all(r.state == FINISHED for r in e.reqs.values()):
            break
    assert all(r.state == FINISHED for r in e.reqs.values())
    assert sum(r["n_evicted"] for r in e.round_log) > 0
    segs = e.poll()
    by = {}
    for s in sorted(segs, key=lambda s: (s["request_id"], s["k"])):
        by.setdefault(s["request_id"], []).extend(s["tokens"])
    assert all(by[rid] == r.script for rid, r in e.reqs.items())
