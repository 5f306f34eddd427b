"""Shared prompt prefixes (DESIGN reading R-PFX) in the oracle:
page accounting pins (P8 extended), reservation of own pages only, and exactness of KV
sharing (a prefixed request computes the same logits as the same prompt without sharing)."""
import numpy as np
import pytest

from oracle.engine import OracleEngine, OracleError, FINISHED, ceil_div
from oracle.model import OracleModel
from synth import engine_params, MODEL_SHAPES, compose_workload


def mk(v, model=None, **kw):
    p = engine_params("paper-4090", **kw)
    return OracleEngine(p, v.tok_skill, v.tok_exec_min_us, v.eos_id, v.vocab, model=model)


PFX = [7 + (i * 13) % 300 for i in range(32)]   # 2 pages


def test_prefix_pages_popped_first_and_never_freed(tiny_vocab):
    e = mk(tiny_vocab, max_ctx=128, n_pages=16, max_batch=4, max_tasks=8)
    assert e.register_prefix(PFX) == 0
    assert sorted(e.prefixes[0]["pages"]) == [0, 1] and e.prefixes[0]["pages"] == [0, 1]
    a = e.submit(0, PFX + [3, 4, 5], 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5] * 4)
    b = e.submit(1, PFX + [9] * 20, 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5] * 4)
    c = e.submit(2, [1, 2, 3], 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5] * 4)      # no prefix
    assert (e.reqs[a].npfx, e.reqs[b].npfx, e.reqs[c].npfx) == (2, 2, 0)
    e.step()
    tabs = e.page_tables()
    # own pages pop in admission order after the prefix's: a needs 1 (35 tokens -> 3 - 2),
    # b needs 2 (52 tokens -> 4 - 2), c needs 1
    assert tabs[a] == [0, 1, 2] and tabs[b] == [0, 1, 3, 4] and tabs[c] == [5]
    log = e.round_log[-1]
    assert log["popped"] == [(a, 2), (b, 3), (b, 4), (c, 5)]
    e.run_until_idle()
    assert all(r.state == FINISHED for r in e.reqs.values())
    # P8 with prefixes: free + prefix pages = pool, the prefix's pages never return
    assert sorted(e.free + e.prefixes[0]["pages"]) == list(range(16))
    assert 0 not in e.free and 1 not in e.free


def test_prefix_invariants_through_a_workload(tiny_vocab):
    v = tiny_vocab
    e = mk(v, max_ctx=256, n_pages=64, max_batch=4, max_tasks=64)
    e.register_prefix(PFX)
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, 0, v, prompt_len_range=(40, 64), max_requests=12)
    for r in reqs:
        e.submit(r.agent_id, PFX + list(r.prompt), r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, 0,
                 script=r.plan)
    for _ in range(10000):
        info = e.step()
        own = sum(len(r.pages) - r.npfx for r in e.reqs.values() if r.holder)
        assert len(e.free) + own + 2 == 64
        for r in e.reqs.values():
            if r.holder:
                assert r.pages[:2] == [0, 1]
                assert len(r.pages) == ceil_div(r.ctx, 16)
        assert sum(r.R - len(r.pages) for r in e.reqs.values() if r.holder) <= len(e.free)
        if info["n_running"] == 0 and all(x.state == FINISHED for x in e.reqs.values()):
            break
    assert sorted(e.free) == list(range(2, 64))


def test_prefix_reservation_counts_own_pages_only(tiny_vocab):
    # pool 8: the prefix takes 2, 6 free.  a = 32 + 80 prompt tokens + 4 new: R = 8 pages in
    # total (more than the 6 free) but 6 own -> admitted; b then needs 1 own page -> refused.
    e = mk(tiny_vocab, max_ctx=128, n_pages=8, max_batch=4, max_tasks=8)
    e.register_prefix(PFX)
    a = e.submit(0, PFX + [3] * 80, 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5] * 4)
    b = e.submit(1, PFX + [4] * 4, 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5] * 4)
    assert e.reqs[a].R == 8 and e.reqs[a].npfx == 2
    info = e.step()
    assert info["n_admitted"] == 1 and info["n_refused_mem"] == 1
    assert e.page_tables()[a] == [0, 1, 2, 3, 4, 5, 6, 7][:7]   # prefix 0, 1 + 5 prompt pages


def test_prefix_validation(tiny_vocab):
    e = mk(tiny_vocab, max_ctx=128, n_pages=4, max_batch=4, max_tasks=8)
    with pytest.raises(OracleError):
        e.register_prefix(PFX[:20])                     # not a multiple of 16
    with pytest.raises(OracleError):
        e.register_prefix([1] * 80)                     # 5 pages > pool of 4
    e.register_prefix(PFX)
    rid = e.submit(0, PFX, 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5])   # equal to the prefix: no share
    assert e.reqs[rid].npfx == 0


def test_prefix_sharing_is_exact_on_the_model(tiny_vocab):
    """KV of a position depends only on the tokens up to it, so sharing a prefix computed
    once gives the same logits as prefilling the whole prompt (pin: a construction)."""
    shape = MODEL_SHAPES["tiny"]
    v = tiny_vocab
    prompt = PFX + [11, 12, 13, 14, 15]
    outs = []
    for share in (False, True):
        e = mk(v, model=OracleModel(shape, seed=3), max_ctx=128, n_pages=16, max_batch=4, max_tasks=8)
        if share:
            e.register_prefix(PFX)
        e.submit(0, prompt, 0, 10 ** 6, -2.0, 1.0, 0, 0, script=[5, 6, 7])
        lg = []
        for _ in range(3):
            e.step()
            lg.append(np.stack(list(e.round_log[-1]["logits"].values())))
        outs.append(np.concatenate(lg))
    assert np.abs(outs[0] - outs[1]).max() < 1e-9
