"""End-to-end parity of the C-ABI engine (rt_submit_request / rt_step /
rt_poll_segment) against the oracle round loop (run on a B200).

* scheduling parity — bit-exact admission order, batch slots, emitted tokens,
  segment records, page tables and free stack, every round (scripted streams,
  SURVEY AMB-17), across policies, per-round admission caps {1, 4, inf} (AMB-8),
  memory pressure, WCET gating and the WALL clock replayed from its log;
* model parity on the tiny C1 model — logits (end-to-end, gated 1e-2) and the
  per-op attention of the capture layer on the GPU's own q and KV pages;
* 8B-shaped operating point — sampled per-op attention and logits checks.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.engine import OracleEngine, FINISHED          # noqa: E402
from oracle.model import OracleModel, paged_attention     # noqa: E402
from oracle import weights as OW                          # noqa: E402
from oracle.bf16 import bf16                              # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params, compose_workload  # noqa: E402
from synth.configs import POLICY_FCFS, POLICY_EDF, CLOCK_WALL, SEG_STREAM, SEG_NONE  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2412_18695_b200 import rt as _rt
    _rt.lib()
    return _rt


def make_pair(rt, vocab, params, shape=None, seed=0, flags=0, model=False, **kw):
    eng = rt.Engine(shape, params, vocab, seed=seed, flags=flags, **kw)
    om = OracleModel(shape, seed=seed) if model else None
    ora = OracleEngine(params, vocab.tok_skill, vocab.tok_exec_min_us, vocab.eos_id, vocab.vocab, model=om)
    return eng, ora


def submit_both(eng, ora, reqs, scripted=True):
    for r in reqs:
        a = eng.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us,
                       len(r.plan), script=r.plan if scripted else None)
        b = ora.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us,
                       len(r.plan), script=r.plan if scripted else None)
        assert a == b


def lockstep(eng, ora, max_rounds=5000, now=None, check_every=1):
    n = 0
    while n < max_rounds:
        t = None if now is None else now(n)
        ig = eng.step(t or 0)
        io = ora.step(t)
        n += 1
        for key in ("t_us", "n_waiting", "n_running", "n_admitted", "n_refused_mem", "n_refused_wcet"):
            assert ig[key] == io[key], (n, key, ig, io)
        if io["n_running"]:
            lg = eng.round_log()
            lo = ora.round_log[-1]
            assert lg["slots"] == lo["slots"], n
            assert lg["admitted"] == lo["admitted"], n
            assert lg["tokens"] == lo["tokens"], n
            assert lg["free"] == lo["free"], n
            if n % check_every == 0:
                assert eng.page_tables() == ora.page_tables(), n
                li = eng.last_round()
                assert li["n_stopped"] == io["n_stopped"] and li["round_us"] == io["round_us"], (li, io)
        if io["n_running"] == 0 and all(r.state == FINISHED for r in ora.reqs.values()):
            break
    sg, so = eng.poll(), ora.poll()
    assert sg == so
    from paper_2412_18695_b200 import rt as _rt
    fs = eng.dump(_rt.RT_DUMP_FREE_STACK, np.int32)
    assert list(fs) == ora.free
    return n, sg


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_sched_parity_c1(rt, seed):
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=4, max_tasks=64, max_ctx=256, n_pages=64)
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, seed, v, prompt_len_range=(40, 64), max_requests=12)
    eng, ora = make_pair(rt, v, p)
    submit_both(eng, ora, reqs)
    n, segs = lockstep(eng, ora)
    assert len({s["request_id"] for s in segs if s["reason"] in (1, 2)}) == 12


def test_poll_ready_pipelined(rt):
    """rt_poll_segment_ready (the non-blocking drain of the pipelined serving loop, bench.py
    e2e): after rt_step of round r returns, every record of rounds <= r - 1 is visible; what it
    returns is always a prefix of the oracle's record sequence (round order, slot order), never
    a partial record; the final blocking poll completes the sequence bit-exact."""
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=16, max_tasks=1024, max_ctx=256, n_pages=96,
                      max_admit_per_round=1 << 30)
    reqs = compose_workload(64, 8.0, 16, range(1, 12), 6.0, 3, v, prompt_len_range=(20, 120), max_requests=300)
    eng, ora = make_pair(rt, v, p)
    submit_both(eng, ora, reqs)
    got, want, through = [], [], [0]
    for n in range(20000):
        eng.step()
        io = ora.step()
        want += ora.poll()
        through.append(len(want))              # records of rounds <= n
        got += eng.poll(wait=False)
        assert len(got) >= through[n], (n, len(got), through[n])   # rounds <= n - 1 all visible
        assert got == want[:len(got)], n
        if io["n_running"] == 0 and all(r.state == FINISHED for r in ora.reqs.values()):
            break
    got += eng.poll()
    assert got == want and len(want) > 100


@pytest.mark.parametrize("policy,max_admit", [(0, 1), (0, 4), (0, 1 << 30), (POLICY_FCFS, 1 << 30),
                                              (POLICY_EDF, 2)])
def test_sched_parity_contention(rt, policy, max_admit):
    # 64 agents, bursty arrivals, small pool (memory refusals), batch 16
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=16, max_tasks=1024, max_ctx=256, n_pages=96, policy=policy,
                      max_admit_per_round=max_admit)
    reqs = compose_workload(64, 8.0, 16, range(1, 12), 6.0, 5, v, prompt_len_range=(20, 120), max_requests=600)
    eng, ora = make_pair(rt, v, p)
    submit_both(eng, ora, reqs)
    n, segs = lockstep(eng, ora, max_rounds=20000, check_every=3)
    assert any(r["n_refused_mem"] > 0 for r in ora.round_log)


@pytest.mark.parametrize("policy,seg_mode", [(POLICY_FCFS, SEG_NONE), (POLICY_FCFS, SEG_STREAM),
                                             (0, SEG_STREAM), (POLICY_EDF, SEG_NONE)])
def test_sched_parity_comparison_systems(rt, policy, seg_mode):
    """SURVEY NEXT-3 on the device scheduler: vLLM (FCFS, no segmentation), vLLM-stream
    (segments delivered, generation never suspended), both without the WCET gate, bit-exact
    against the oracle every round on a contended trace (memory refusals, arm plans > 16
    tokens so NONE-mode records exceed the method's 10-token cap)."""
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=16, max_tasks=1024, max_ctx=256, n_pages=96, policy=policy,
                      seg_mode=seg_mode, wcet_off=1)
    reqs = compose_workload(64, 8.0, 16, range(1, 12), 6.0, 7, v, prompt_len_range=(20, 120), max_requests=400)
    eng, ora = make_pair(rt, v, p)
    submit_both(eng, ora, reqs)
    n, segs = lockstep(eng, ora, max_rounds=20000, check_every=3)
    if seg_mode == SEG_NONE:
        assert any(s["tok_end"] - s["tok_begin"] > 16 for s in segs)
    admits = [a for r in ora.round_log for a in r["admitted"]]
    assert len(admits) == len(set(admits)) == len(reqs)   # never suspended / re-queued


@pytest.mark.parametrize("name", ["c5", "c4"])
def test_sched_parity_at_c4_c5_task_counts(rt, name):
    """Scheduling-only parity at the task counts of BASELINE configs[3-4] (the bench's CPU
    replays): C5 = 512 agents of long robot-arm plans (160 tokens, max_new 256), 128-token
    prompts, AMB-26 reservations on a pool that refuses admissions, batch 512; C4 = 1024 agents
    of traces 1-11, batch 128.  Hundreds of waiting candidates per round exercise the device
    sorts (rank sort <= 128, register bitonic <= 1024, shared-memory bitonic beyond) and the
    closed-form admission; rounds, admissions, segments, page tables and the free stack are
    bit-exact against the oracle."""
    v = make_vocab(128256)
    if name == "c5":
        p = engine_params("b200-roofline", max_batch=512, max_tasks=2048, max_ctx=4096, n_pages=277 * 24)
        reqs = compose_workload(512, 64.0, 16, range(9, 12), 10.0, 0, v, prompt_len_range=(128, 128),
                                max_requests=1536, plan_len=160)
    else:
        p = engine_params("b200-roofline", max_batch=128, max_tasks=2048, max_ctx=4096, n_pages=1 << 16)
        reqs = compose_workload(1024, 640.0, 16, range(1, 12), 10.0, 0, v, prompt_len_range=(64, 64),
                                max_requests=2000)
    eng, ora = make_pair(rt, v, p)
    for r in reqs:
        mx = 256 if name == "c5" else len(r.plan)
        a = eng.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, mx,
                       script=r.plan)
        b = ora.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, mx,
                       script=r.plan)
        assert a == b
    n, segs = lockstep(eng, ora, max_rounds=400, check_every=20)
    waiting = max(r["n_waiting"] for r in ora.round_log)
    assert waiting > 128                      # beyond the rank sort
    if name == "c5":
        assert any(r["n_refused_mem"] > 0 for r in ora.round_log)
    else:
        assert waiting > 1024                 # the shared-memory bitonic path
    eng.close()


def _evict_workload(v, **kw):
    p = engine_params("paper-4090", max_batch=8, max_tasks=512, max_ctx=256, n_pages=40, host_pages=64,
                      swap_us_per_page=116, **kw)
    reqs = compose_workload(24, 6.0, 8, range(1, 12), 8.0, 9, v, prompt_len_range=(20, 90), max_requests=120)
    return p, reqs


def test_sched_parity_kv_eviction(rt):
    """NEXT-2 on the device scheduler (R-EVICT): the same contended trace as the oracle pin
    (tests/test_oracle_evict.py) — evictions / restores per round, page tables, host page
    tables, free stack and host free stack bit-exact every round."""
    v = make_vocab(512)
    p, reqs = _evict_workload(v)
    eng, ora = make_pair(rt, v, p)
    submit_both(eng, ora, reqs)
    n_ev = 0
    for n in range(20000):
        ig, io = eng.step(), ora.step()
        for key in ("t_us", "n_running", "n_admitted", "n_refused_mem"):
            assert ig[key] == io[key], (n, key, ig, io)
        assert (ig["n_evicted"], ig["n_restored"]) == (io.get("n_evicted", 0), io.get("n_restored", 0)), n
        n_ev += io.get("n_evicted", 0)
        if io["n_running"]:
            assert eng.round_log()["slots"] == ora.round_log[-1]["slots"], n
        assert eng.page_tables() == ora.page_tables(), n
        assert eng.host_page_tables() == ora.host_page_tables(), n
        assert list(eng.dump(rt.RT_DUMP_HOST_FREE_STACK, np.int32)) == ora.hfree, n
        if io["n_running"] == 0 and all(r.state == FINISHED for r in ora.reqs.values()):
            break
    assert n_ev > 0
    assert eng.poll() == ora.poll()
    assert list(eng.dump(rt.RT_DUMP_FREE_STACK, np.int32)) == ora.free


def test_tiny_model_kv_eviction_e2e(rt):
    """KV evicted to pinned host pages and restored (no re-prefill) keeps the model exact:
    C1-shaped tiny model under the eviction workload, logits of every round against the
    oracle (whose KV never moves) and the segment stream bit-exact."""
    shape = MODEL_SHAPES["tiny"]
    v = make_vocab(shape.vocab)
    p, reqs = _evict_workload(v)
    eng, ora = make_pair(rt, v, p, shape=shape, seed=5, flags=rt.RT_FLAG_KEEP_LOGITS, model=True)
    submit_both(eng, ora, reqs[:60])
    worst = 0.0
    n_ev = n_rs = 0
    for n in range(20000):
        ig, io = eng.step(), ora.step()
        assert ig["n_running"] == io["n_running"] and ig["n_evicted"] == io.get("n_evicted", 0), n
        n_ev += ig["n_evicted"]
        n_rs += ig["n_restored"]
        if io["n_running"]:
            B = io["n_running"]
            lg = eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(B, -1)
            lo = np.stack([ora.round_log[-1]["logits"][rid] for rid in ora.round_log[-1]["slots"]])
            worst = max(worst, float(np.abs(lg - lo).max()))
        if io["n_running"] == 0 and all(r.state == FINISHED for r in ora.reqs.values()):
            break
    assert n_ev > 0 and n_rs > 0
    assert worst < 1e-2, worst
    assert eng.poll() == ora.poll()


def test_sched_parity_wcet_gate(rt):
    # slow paper-4090 clock with gamma: urgent running tasks block admissions (WCET)
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=8, max_tasks=128, max_ctx=256, n_pages=256)
    reqs = compose_workload(32, 4.0, 8, [6, 7, 8, 1, 2], 4.0, 11, v, prompt_len_range=(10, 30))
    eng, ora = make_pair(rt, v, p)
    submit_both(eng, ora, reqs)
    lockstep(eng, ora, max_rounds=20000, check_every=5)
    assert any(r["n_refused_wcet"] > 0 for r in ora.round_log)


def test_sched_parity_wall_clock_replay(rt):
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=4, max_tasks=64, max_ctx=256, n_pages=64, clock_mode=CLOCK_WALL)
    reqs = compose_workload(8, 2.0, 4, range(1, 9), 3.0, 4, v, prompt_len_range=(8, 40))
    eng, ora = make_pair(rt, v, p)
    submit_both(eng, ora, reqs)
    rng = np.random.default_rng(0)
    clock = np.cumsum(rng.integers(5000, 40000, 20000))     # recorded wall-clock log
    lockstep(eng, ora, max_rounds=20000, now=lambda i: int(clock[i]), check_every=4)


def test_round_exchange_single_rank_nccl(rt):
    """a12 on hardware: the per-round ncclAllGather + device merge (1-rank communicator,
    RT_FLAG_FORCE_EXCHANGE) yields exactly the oracle's top-16 (Pri, arrival, id) keys."""
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=8, max_tasks=512, max_ctx=256, n_pages=96)
    reqs = compose_workload(64, 8.0, 16, range(1, 12), 3.0, 9, v, prompt_len_range=(20, 100), max_requests=300)
    eng, ora = make_pair(rt, v, p, flags=rt.RT_FLAG_FORCE_EXCHANGE)
    submit_both(eng, ora, reqs)
    checked = 0
    for n in range(3000):
        ig, io = eng.step(), ora.step()
        assert ig["n_running"] == io["n_running"]
        if io["n_running"] == 0:
            if all(r.state == FINISHED for r in ora.reqs.values()):
                break
            continue
        merged = eng.dump(rt.RT_DUMP_MERGED, np.float64).reshape(16, 4)
        exp = ora.round_log[-1]["topk"]
        got = [tuple(m) for m in merged if m[2] >= 0]
        assert len(got) == len(exp), n
        for g, e in zip(got, exp):
            assert g[0] == e[0] and g[1] == e[1] and g[2] == e[2] and g[3] == e[3], (n, g, e)
        checked += int(len(exp) > 1)
    assert checked > 20


def test_submit_errors(rt):
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=4, max_tasks=2, max_ctx=64, n_pages=2)
    eng = rt.Engine(None, p, v)
    with pytest.raises(rt.RtError) as ex:
        eng.submit(0, [1], 0, 10, 0.5, 1.0, 0, script=[5])
    assert ex.value.code == rt.RT_E_INVAL
    with pytest.raises(rt.RtError) as ex:
        eng.submit(0, [1] * 40, 0, 10, -1.0, 1.0, 0, script=[5])
    assert ex.value.code == rt.RT_E_NOMEM
    with pytest.raises(rt.RtError) as ex:
        eng.submit(0, [1], 0, 10, -1.0, 1.0, 0)                  # no model -> needs a script
    assert ex.value.code == rt.RT_E_INVAL
    eng.submit(0, [1], 0, 10, -1.0, 1.0, 0, script=[5])
    eng.submit(0, [1], 0, 10, -1.0, 1.0, 0, script=[5])
    with pytest.raises(rt.RtError) as ex:
        eng.submit(0, [1], 0, 10, -1.0, 1.0, 0, script=[5])      # table full until polled
    assert ex.value.code == rt.RT_E_NOMEM
    eng.step()
    assert len(eng.poll()) == 2
    eng.submit(0, [1], 0, 10, -1.0, 1.0, 0, script=[5])          # slots recycled after poll


# ------------------------------------------------------------- model parity
def test_tiny_model_chunked_forward(rt):
    """Prefill rounds larger than one forward chunk (max_rows_per_forward = 48: the 4 x 40-64
    prompt rows of the first rounds run as 3-6 chunks): chunk 0's embedding is the one launched
    before the plan handshake (k_embed_plan, row count read on the device), the others the
    per-chunk k_embed; logits end to end vs the oracle and bit-exact segments."""
    shape = MODEL_SHAPES["tiny"]
    v = make_vocab(shape.vocab)
    p = engine_params("paper-4090", max_batch=4, max_tasks=64, max_ctx=256, n_pages=64)
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, 4, v, prompt_len_range=(40, 64), max_requests=12)
    eng, ora = make_pair(rt, v, p, shape=shape, seed=5, flags=rt.RT_FLAG_KEEP_LOGITS, model=True,
                         max_rows_per_forward=48)
    submit_both(eng, ora, reqs)
    worst, chunked = 0.0, 0
    for n in range(400):
        ig, io = eng.step(), ora.step()
        assert ig["n_running"] == io["n_running"] and ig["n_rows"] == io.get("n_rows", ig["n_rows"])
        chunked += ig["n_rows"] > 48
        if io["n_running"] == 0:
            if all(r.state == FINISHED for r in ora.reqs.values()):
                break
            continue
        lg = eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(io["n_running"], -1)
        lo = np.stack([ora.round_log[-1]["logits"][rid] for rid in ora.round_log[-1]["slots"]])
        worst = max(worst, float(np.abs(lg - lo).max()))
    assert chunked > 0
    assert eng.poll() == ora.poll()
    assert worst <= 1e-2, worst


@pytest.mark.parametrize("gemm_path", [0, 1, 2, 3])
def test_tiny_model_e2e_and_per_op(rt, gemm_path):
    """C1 end to end against the oracle, through every projection kernel path (rt_config.gemm_path:
    the measured dispatch, split-K / one tile per CTA, hybrid stream-K, CTA pairs — the prefill
    rounds' N > 128 rows take the forced path wherever it applies)."""
    shape = MODEL_SHAPES["tiny"]
    v = make_vocab(shape.vocab)
    p = engine_params("paper-4090", max_batch=4, max_tasks=64, max_ctx=256, n_pages=64)
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, 0, v, prompt_len_range=(40, 64), max_requests=12)
    flags = rt.RT_FLAG_KEEP_LOGITS | rt.RT_FLAG_CAPTURE
    eng, ora = make_pair(rt, v, p, shape=shape, seed=3, flags=flags, model=True, capture_layer=1,
                         gemm_path=gemm_path)
    submit_both(eng, ora, reqs)
    worst_logit = worst_attn = worst_lm = 0.0
    lm = OW.matrix(3, OW.TID_LM, range(shape.vocab), shape.d_model)
    for n in range(400):
        ig, io = eng.step(), ora.step()
        assert ig["n_running"] == io["n_running"]
        if io["n_running"] == 0:
            if all(r.state == FINISHED for r in ora.reqs.values()):
                break
            continue
        B = io["n_running"]
        lg = eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(B, -1)
        lo = np.stack([ora.round_log[-1]["logits"][rid] for rid in ora.round_log[-1]["slots"]])
        worst_logit = max(worst_logit, float(np.abs(lg - lo).max()))
        # logits per op: oracle lm_head on the GPU's own final bf16 hidden
        hid = eng.dump(rt.RT_DUMP_HIDDEN, np.uint16).reshape(B, -1)
        h = (hid.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        worst_lm = max(worst_lm, float(np.abs(h @ lm.T - lg).max()))
        # attention per op (capture layer): oracle attention on the GPU's q and pages
        rows = eng.dump(rt.RT_DUMP_ROWS, np.int32).reshape(-1, 3)
        q = eng.dump(rt.RT_DUMP_CAPTURE_Q, np.float32).reshape(len(rows), shape.n_q_heads, shape.head_dim)
        o = eng.dump(rt.RT_DUMP_CAPTURE_O, np.float32).reshape(len(rows), shape.n_q_heads, shape.head_dim)
        kv = eng.dump(rt.RT_DUMP_KV_LAYER, np.uint16).reshape(p.n_pages, 2, shape.n_kv_heads, 16, shape.head_dim)
        kvf = (kv.astype(np.uint32) << 16).view(np.float32)
        kp = kvf[:, 0].transpose(0, 2, 1, 3)
        vp = kvf[:, 1].transpose(0, 2, 1, 3)
        tabs = eng.dump(rt.RT_DUMP_PAGE_TABLES, np.int32).reshape(p.max_tasks, -1)
        for i in range(0, len(rows), max(1, len(rows) // 16)):
            task, pos, _ = rows[i]
            ref = paged_attention(q[i], kp, vp, tabs[task], pos + 1)
            worst_attn = max(worst_attn, float(np.abs(o[i] - ref).max()))
    assert worst_attn < 6e-3, worst_attn
    assert worst_lm < 1e-3, worst_lm
    assert worst_logit < 1e-2, worst_logit
    assert eng.poll() == ora.poll()


def test_tiny_model_free_running_tokens(rt):
    """Free-running greedy: GPU argmax stream fed to the oracle (teacher forcing,
    AMB-17); argmax must agree wherever the oracle's top-2 margin exceeds 2x drift."""
    shape = MODEL_SHAPES["tiny"]
    v = make_vocab(shape.vocab)
    p = engine_params("paper-4090", max_batch=4, max_tasks=16, max_ctx=256, n_pages=64)
    eng = rt.Engine(shape, p, v, seed=5, flags=rt.RT_FLAG_KEEP_LOGITS)
    om = OracleModel(shape, seed=5)
    rng = np.random.default_rng(1)
    prompts = [rng.integers(0, 400, 30 + 7 * i) for i in range(3)]
    for i, pr in enumerate(prompts):
        eng.submit(i, pr, 0, 1_000_000, -2.0, 1.0, 0, 24)
    seqs = {i: list(map(int, pr)) for i, pr in enumerate(prompts)}
    agree = checked = 0
    for _ in range(60):
        info = eng.step()
        if info["n_running"] == 0:
            break
        lg = eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(info["n_running"], -1)
        log = eng.round_log()
        for s, rid in enumerate(log["slots"]):
            ref_rows = [(rid + 100, j, t) for j, t in enumerate(seqs[rid])]
            om.drop(rid + 100)
            ref = om.logits(om.forward(ref_rows)[-1:])[0]
            top2 = np.sort(ref)[-2:]
            drift = float(np.abs(lg[s] - ref).max())
            if top2[1] - top2[0] > 2 * drift:
                checked += 1
                agree += int(np.argmax(ref) == log["tokens"][s])
            seqs[rid].append(log["tokens"][s])
    assert checked > 10 and agree == checked


def _sampled_checks(rt, eng, shape, p, seed, n_rows_check=8, n_vocab=512):
    rows = eng.dump(rt.RT_DUMP_ROWS, np.int32).reshape(-1, 3)
    nq, nkv, hd = shape.n_q_heads, shape.n_kv_heads, shape.head_dim
    q = eng.dump(rt.RT_DUMP_CAPTURE_Q, np.float32).reshape(len(rows), nq, hd)
    o = eng.dump(rt.RT_DUMP_CAPTURE_O, np.float32).reshape(len(rows), nq, hd)
    kv = eng.dump(rt.RT_DUMP_KV_LAYER, np.uint16).reshape(p.n_pages, 2, nkv, 16, hd)
    tabs = eng.dump(rt.RT_DUMP_PAGE_TABLES, np.int32).reshape(p.max_tasks, -1)
    rng = np.random.default_rng(seed)
    worst = 0.0
    for i in rng.choice(len(rows), min(n_rows_check, len(rows)), replace=False):
        task, pos, _ = rows[i]
        npg = (pos + 16) // 16
        pages = tabs[task][:npg]
        kvf = (kv[pages].astype(np.uint32) << 16).view(np.float32)
        kp, vp = kvf[:, 0].transpose(0, 2, 1, 3), kvf[:, 1].transpose(0, 2, 1, 3)
        ref = paged_attention(q[i], kp, vp, list(range(npg)), pos + 1)
        worst = max(worst, float(np.abs(o[i] - ref).max()))
    B = eng.last_round()["n_running"]
    lg = eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(B, -1)
    hid = eng.dump(rt.RT_DUMP_HIDDEN, np.uint16).reshape(B, -1)
    h = (hid.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    cols = np.concatenate([rng.choice(shape.vocab, n_vocab, replace=False), np.argmax(lg, axis=1)])
    W = OW.matrix(seed, OW.TID_LM, cols, shape.d_model)
    lerr = float(np.abs(h @ W.T - lg[:, cols]).max())
    return worst, lerr


def test_c3_mixed_256_shape_sampled(rt):
    """BASELINE configs[2] shape: 256 mixed drone / robot-arm agents (prompts 1300 / 2884),
    8B layer dims with 4 layers (the decode GEMMs run at N = 256, the BN = 256 path)."""
    from synth.configs import ModelShape
    s8 = MODEL_SHAPES["llama3-8b"]
    shape = ModelShape("c3", 4, s8.d_model, s8.n_q_heads, s8.n_kv_heads, s8.head_dim, s8.d_ff, s8.vocab)
    v = make_vocab(shape.vocab)
    p = engine_params("b200-roofline", max_batch=256, max_tasks=512, max_ctx=3072, n_pages=256 * 186)
    flags = rt.RT_FLAG_KEEP_LOGITS | rt.RT_FLAG_CAPTURE
    eng = rt.Engine(shape, p, v, seed=13, flags=flags, capture_layer=3, max_rows_per_forward=8192)
    from synth.traces import make_trace
    for a in range(256):
        tid = (a % 8) + 1 if a % 2 == 0 else 9 + (a % 3)
        tr = make_trace(tid, v, seed=a)
        eng.submit(a, tr.prompt, 0, tr.ert_us, tr.alpha, tr.beta, 90000, script=tr.plan)
    for _ in range(30):
        info = eng.step()
        if info["n_running"] == 256 and info["n_prefill_rows"] == 0:
            break
    assert info["n_running"] == 256 and info["n_prefill_rows"] == 0
    worst, lerr = _sampled_checks(rt, eng, shape, p, 13)
    assert worst < 6e-3, worst
    assert lerr < 1e-2, lerr


def test_llama70b_dims_sampled(rt):
    """BASELINE configs[4] layer dims (d 8192, 64 / 8 heads: G = 8, ff 28672), 2 layers,
    128 running requests with short unique prompts (C5 plans)."""
    from synth.configs import ModelShape
    s70 = MODEL_SHAPES["llama3-70b"]
    shape = ModelShape("c5", 2, s70.d_model, s70.n_q_heads, s70.n_kv_heads, s70.head_dim, s70.d_ff, s70.vocab)
    v = make_vocab(shape.vocab)
    p = engine_params("b200-roofline", max_batch=128, max_tasks=256, max_ctx=512, n_pages=128 * 32)
    flags = rt.RT_FLAG_KEEP_LOGITS | rt.RT_FLAG_CAPTURE
    eng = rt.Engine(shape, p, v, seed=17, flags=flags, capture_layer=1, max_rows_per_forward=8192)
    rng = np.random.default_rng(5)
    from synth.traces import make_trace
    for a in range(128):
        tr = make_trace(9 + a % 3, v, seed=a, prompt_len=int(rng.integers(100, 160)), plan_len=150)
        eng.submit(a, tr.prompt, 0, tr.ert_us, tr.alpha, tr.beta, 90000, script=tr.plan)
    for _ in range(30):
        info = eng.step()
        if info["n_running"] == 128 and info["n_prefill_rows"] == 0:
            break
    assert info["n_running"] == 128
    worst, lerr = _sampled_checks(rt, eng, shape, p, 17)
    assert worst < 6e-3, worst
    assert lerr < 1e-2, lerr


def test_llama8b_shape_sampled(rt):
    """BASELINE configs[1] shape (Llama-3-8B dims, random init) at the bench's
    launch configuration: per-op attention on sampled (row, head) pairs and
    logits on sampled vocab rows, computed one by one by the oracle."""
    shape = MODEL_SHAPES["llama3-8b"]
    v = make_vocab(shape.vocab)
    p = engine_params("b200-roofline", max_batch=64, max_tasks=128, max_ctx=2048, n_pages=64 * 90)
    flags = rt.RT_FLAG_KEEP_LOGITS | rt.RT_FLAG_CAPTURE
    eng = rt.Engine(shape, p, v, seed=11, flags=flags, capture_layer=31, max_rows_per_forward=4096)
    reqs = compose_workload(64, 100.0, 64, range(1, 9), 0.2, 2, v, prompt_len_range=(1250, 1310), max_requests=64)
    for r in reqs:
        eng.submit(r.agent_id, r.prompt, 0, r.ert_us, r.alpha, r.beta, r.exec_window_us, 0, script=r.plan)
    # after the 82k-token prefill round the WCET speed window (5 rounds) briefly gates
    # resumes; run until every request is back in the batch
    for _ in range(20):
        info = eng.step()
        if info["n_running"] == 64 and info["n_prefill_rows"] == 0:
            break
    B = info["n_running"]
    assert B == 64 and info["n_prefill_rows"] == 0
    rows = eng.dump(rt.RT_DUMP_ROWS, np.int32).reshape(-1, 3)
    nq, nkv, hd = shape.n_q_heads, shape.n_kv_heads, shape.head_dim
    q = eng.dump(rt.RT_DUMP_CAPTURE_Q, np.float32).reshape(len(rows), nq, hd)
    o = eng.dump(rt.RT_DUMP_CAPTURE_O, np.float32).reshape(len(rows), nq, hd)
    kv = eng.dump(rt.RT_DUMP_KV_LAYER, np.uint16).reshape(p.n_pages, 2, nkv, 16, hd)
    tabs = eng.dump(rt.RT_DUMP_PAGE_TABLES, np.int32).reshape(p.max_tasks, -1)
    rng = np.random.default_rng(0)
    worst = 0.0
    for i in rng.choice(len(rows), 8, replace=False):
        task, pos, _ = rows[i]
        npg = (pos + 16) // 16
        pages = tabs[task][:npg]
        kvf = (kv[pages].astype(np.uint32) << 16).view(np.float32)
        kp, vp = kvf[:, 0].transpose(0, 2, 1, 3), kvf[:, 1].transpose(0, 2, 1, 3)
        ref = paged_attention(q[i], kp, vp, list(range(npg)), pos + 1)
        worst = max(worst, float(np.abs(o[i] - ref).max()))
    assert worst < 6e-3, worst
    lg = eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(B, -1)
    hid = eng.dump(rt.RT_DUMP_HIDDEN, np.uint16).reshape(B, -1)
    h = (hid.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    cols = np.concatenate([rng.choice(shape.vocab, 512, replace=False), np.argmax(lg, axis=1)])
    W = OW.matrix(11, OW.TID_LM, cols, shape.d_model)
    err = np.abs(h @ W.T - lg[:, cols]).max()
    assert err < 1e-2, err


def test_device_trace_records(rt):
    """RT_FLAG_TRACE: one record per CTA with ordered timestamps, every kernel role present."""
    shape = MODEL_SHAPES["tiny"]
    v = make_vocab(shape.vocab)
    p = engine_params("paper-4090", max_batch=4, max_tasks=16, max_ctx=256, n_pages=64)
    eng = rt.Engine(shape, p, v, seed=5, flags=rt.RT_FLAG_TRACE)
    for i in range(3):
        eng.submit(i, [1 + i, 2, 3, 4], 0, 1_000_000, -1.0, 1.0, 0, max_new_tokens=8)
    eng.step()
    eng.reset_stats()
    for _ in range(3):
        eng.step()
    eng.sync()
    tr = eng.trace()
    assert len(tr) > 0
    tr = tr[(tr["kind"] & 0x80) == 0]   # phase records carry cycle counts, not timestamps
    assert (tr["t_entry"] <= tr["t_ready"]).all() and (tr["t_ready"] <= tr["t_exit"]).all()
    kinds = set(int(k) & 0xFF for k in tr["kind"])
    assert {1, 2, 4, 5, 6, 7, 8} <= kinds, kinds
    gemm = tr[(tr["kind"] & 0xFF) == 1]
    assert (gemm["t_aux"] >= gemm["t_ready"]).all() and (gemm["t_aux"] <= gemm["t_exit"]).all()
    # 3 decode rounds: one launch of the scheduler pre/post kernels each
    grids = {int(k) & 0xFF: set() for k in tr["kind"]}
    for r in tr:
        grids[int(r["kind"]) & 0xFF].add(int(r["grid"]))
    assert len(grids[5]) == 3 and len(grids[6]) == 3
    assert len(grids[2]) > 0 and len(grids[2]) % shape.n_layers == 0
    eng.close()


# ------------------------------------------------------------- shared prefixes (NEXT-1)
PFX = [7 + (i * 13) % 300 for i in range(48)]   # 3 pages


@pytest.mark.parametrize("n_pages", [64, 24])
def test_sched_parity_with_shared_prefix(rt, n_pages):
    """Prefix pages popped at registration, shared read-only by every prefixed request,
    reservations of own pages only: page tables, free stack and segments bit-exact."""
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=4, max_tasks=64, max_ctx=256, n_pages=n_pages)
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, 4, v, prompt_len_range=(20, 64), max_requests=12)
    eng, ora = make_pair(rt, v, p)
    assert eng.register_prefix(PFX) == ora.register_prefix(PFX) == 0
    for i, r in enumerate(reqs):   # two thirds of the requests carry the prefix
        r.prompt = (PFX + list(r.prompt)) if i % 3 else list(r.prompt)
    submit_both(eng, ora, reqs)
    lockstep(eng, ora)
    tabs = eng.dump(rt.RT_DUMP_PAGE_TABLES, np.int32)
    assert sorted(list(eng.dump(rt.RT_DUMP_FREE_STACK, np.int32)) + ora.prefixes[0]["pages"]) == list(range(n_pages))


def test_tiny_model_shared_prefix_parity(rt):
    """Prefix KV computed once by the registration forward; prefixed requests prefill only
    their own rows: logits and per-op attention vs the oracle."""
    shape = MODEL_SHAPES["tiny"]
    v = make_vocab(shape.vocab)
    p = engine_params("paper-4090", max_batch=4, max_tasks=64, max_ctx=256, n_pages=64)
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, 6, v, prompt_len_range=(20, 40), max_requests=8)
    flags = rt.RT_FLAG_KEEP_LOGITS | rt.RT_FLAG_CAPTURE
    eng, ora = make_pair(rt, v, p, shape=shape, seed=3, flags=flags, model=True, capture_layer=1)
    assert eng.register_prefix(PFX) == ora.register_prefix(PFX)
    for r in reqs:
        r.prompt = PFX + list(r.prompt)
    submit_both(eng, ora, reqs)
    worst_logit = worst_attn = 0.0
    n_pf_rows = 0
    for n in range(400):
        ig, io = eng.step(), ora.step()
        assert ig["n_running"] == io["n_running"]
        if io["n_running"] == 0:
            if all(r.state == FINISHED for r in ora.reqs.values()):
                break
            continue
        n_pf_rows += ig["n_prefill_rows"]
        B = io["n_running"]
        lg = eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(B, -1)
        lo = np.stack([ora.round_log[-1]["logits"][rid] for rid in ora.round_log[-1]["slots"]])
        worst_logit = max(worst_logit, float(np.abs(lg - lo).max()))
        rows = eng.dump(rt.RT_DUMP_ROWS, np.int32).reshape(-1, 3)
        q = eng.dump(rt.RT_DUMP_CAPTURE_Q, np.float32).reshape(len(rows), shape.n_q_heads, shape.head_dim)
        o = eng.dump(rt.RT_DUMP_CAPTURE_O, np.float32).reshape(len(rows), shape.n_q_heads, shape.head_dim)
        kv = eng.dump(rt.RT_DUMP_KV_LAYER, np.uint16).reshape(p.n_pages, 2, shape.n_kv_heads, 16, shape.head_dim)
        kvf = (kv.astype(np.uint32) << 16).view(np.float32)
        kp = kvf[:, 0].transpose(0, 2, 1, 3)
        vp = kvf[:, 1].transpose(0, 2, 1, 3)
        tabs = eng.dump(rt.RT_DUMP_PAGE_TABLES, np.int32).reshape(p.max_tasks, -1)
        for i in range(0, len(rows), max(1, len(rows) // 16)):
            task, pos, _ = rows[i]
            assert pos >= 0
            ref = paged_attention(q[i], kp, vp, tabs[task], pos + 1)
            worst_attn = max(worst_attn, float(np.abs(o[i] - ref).max()))
    # every prefill round computed only the rows after the 48 shared positions
    assert n_pf_rows == sum(len(r.prompt) - 48 for r in reqs)
    assert worst_attn < 6e-3, worst_attn
    assert worst_logit < 1e-2, worst_logit
    assert eng.poll() == ora.poll()


@pytest.mark.parametrize("grammar", [1, 2, 3])
def test_sched_parity_stop_grammars(rt, grammar):
    """NEXT-4 on the device: the DFA / chat stop checker against the oracle's regex over the
    detokenized text, bit-exact segments every round, on
    (a) generated robot plans / chat text and (b) fuzz scripts of random special tokens
    (names, parentheses, digits, ";", words, sentence ends) that exercise every near miss."""
    from synth.grammar import make_grammar_vocab, robot_plan, chat_text
    gv = make_grammar_vocab(512)
    p = engine_params("paper-4090", max_batch=8, max_tasks=256, max_ctx=256, n_pages=256, stop_grammar=grammar,
                      max_seg_tokens=12)
    eng = rt.Engine(None, p, gv)
    ora = OracleEngine(p, gv.tok_skill, gv.tok_exec_min_us, gv.eos_id, gv.vocab, grammar=gv)
    rng = np.random.default_rng(grammar)
    special = [t for t in range(gv.words[1], gv.eos_id)] + list(range(0, 8))
    for i in range(48):
        if i % 2 == 0:
            script = robot_plan(gv, rng, n_stmts=4) if grammar == 1 else chat_text(gv, rng)
        else:
            script = np.array([special[int(x)] for x in rng.integers(0, len(special), 60)] + [gv.eos_id])
        prompt = rng.integers(0, gv.words[1], 20)
        arr = int(i * 20000)
        a = eng.submit(i % 16, prompt, arr, 1_000_000, -2.0, 1.0, 0, len(script), script=script)
        b = ora.submit(i % 16, prompt, arr, 1_000_000, -2.0, 1.0, 0, len(script), script=script)
        assert a == b
    n, segs = lockstep(eng, ora, max_rounds=20000, check_every=7)
    assert sum(1 for s in segs if s["reason"] == 3) > 20


def test_set_timing_toggles_event_stats_only(rt):
    """rt_set_timing (bench pass A / pass B): per-kernel CUDA-event timing on or off does not
    change any result; attention stats accumulate only while it is on."""
    shape = MODEL_SHAPES["tiny"]
    v = make_vocab(shape.vocab)
    p = engine_params("paper-4090", max_batch=4, max_tasks=64, max_ctx=256, n_pages=64)
    reqs = compose_workload(4, 1.0, 2, range(1, 9), 30.0, 2, v, prompt_len_range=(40, 64), max_requests=6)
    outs = []
    for toggle in (False, True):
        eng = rt.Engine(shape, p, v, seed=4, flags=rt.RT_FLAG_TIMING | rt.RT_FLAG_KEEP_LOGITS)
        for r in reqs:
            eng.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, len(r.plan),
                       script=r.plan)
        logits = []
        for i in range(30):
            if toggle:
                eng.set_timing(i % 2 == 0)
            info = eng.step()
            if info["n_running"]:
                logits.append(eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(info["n_running"], -1).copy())
        eng.sync()
        segs = eng.poll()
        if toggle:
            eng.set_timing(False)
            eng.reset_stats()
            for _ in range(3):
                eng.step()
            assert eng.stats()["attn_launches"] == 0
        outs.append((segs, logits))
        eng.close()
    assert outs[0][0] == outs[1][0]
    assert all(np.array_equal(a, b) for a, b in zip(outs[0][1], outs[1][1]))


@pytest.mark.parametrize("gemm_path", [0, 1, 2, 3])
def test_prefill_and_decode_rounds_bitwise_deterministic(rt, gemm_path):
    """Run-to-run determinism of every projection path (the cluster split-K in pull mode once
    let a peer read a half-parked partial tile: logits differed by up to 0.19 between identical
    runs; tools/determinism_check.py): the same scripted rounds twice give bit-identical
    logits."""
    from synth.configs import ModelShape
    from synth.traces import make_trace
    s8 = MODEL_SHAPES["llama3-8b"]
    shape = ModelShape("det", 2, s8.d_model, s8.n_q_heads, s8.n_kv_heads, s8.head_dim, s8.d_ff, s8.vocab)
    v = make_vocab(shape.vocab)
    p = engine_params("b200-roofline", max_batch=8, max_tasks=16, max_ctx=512, n_pages=8 * 32)
    runs = []
    for _ in range(2):
        eng = rt.Engine(shape, p, v, seed=23, flags=rt.RT_FLAG_KEEP_LOGITS, max_rows_per_forward=4096,
                        gemm_path=gemm_path)
        for a in range(8):
            tr = make_trace(1 + a, v, seed=a, prompt_len=64, plan_len=12)
            eng.submit(a, tr.prompt, 0, tr.ert_us, tr.alpha, tr.beta, 90000, script=tr.plan)
        logs = []
        for _ in range(4):
            B = eng.step()["n_running"]
            logs.append(eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(B, -1).copy())
        eng.close()
        runs.append(logs)
    for a, b in zip(*runs):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_sched_parity_c5_slice_retention_stress(rt):
    """SURVEY §8(d) C5 per-GPU slice, scheduling only (BASELINE configs[4]: 4096 agents over 8
    GPUs = 512 per GPU, 70B dims; long robot-arm plans of 160 tokens in >10 segments, 128-token
    prompts, AMB-26 reservations of prompt + 256 new tokens = 24 pages on a pool that holds
    277 of them (the 35 GB left beside 141 GB of weights): admission refusals and long page
    retention.  Device scheduler == oracle every round (admissions, refusals, slots, page
    tables, free stack, segment records)."""
    v = make_vocab(128256)
    p = engine_params("b200-roofline", max_batch=512, max_tasks=2048, max_ctx=512, n_pages=277 * 24)
    reqs = compose_workload(512, 64.0, 16, range(9, 12), 3.0, 7, v, prompt_len_range=(128, 128), plan_len=160,
                            max_requests=900)
    eng, ora = make_pair(rt, v, p)
    for r in reqs:
        a = eng.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, 256,
                       script=r.plan)
        b = ora.submit(r.agent_id, r.prompt, r.arrival_us, r.ert_us, r.alpha, r.beta, r.exec_window_us, 256,
                       script=r.plan)
        assert a == b
    refused = 0
    orig_step = ora.step

    def counting_step(t=None):
        nonlocal refused
        info = orig_step(t)
        refused += info.get("n_refused_mem", 0)
        return info
    ora.step = counting_step
    n, segs = lockstep(eng, ora, max_rounds=20000, check_every=25)
    assert refused > 0                                  # the pool refuses admissions
    assert len({s["request_id"] for s in segs if s["reason"] in (1, 2)}) == len(reqs)
    assert max(s["k"] for s in segs) >= 10              # long multi-segment plans retained


def test_sched_parity_wcet_lag_hand_worked(rt):
    """The hand-worked R-WCET trace (tests/test_oracle_engine.py) on the device scheduler:
    B admitted at round 1 on the pre-admission speed, C refused at round 2, A's segment
    dispatched at 227720 us."""
    v = make_vocab(512)
    p = engine_params("paper-4090", max_batch=4, max_tasks=8, max_ctx=64, n_pages=16, max_admit_per_round=1)
    eng, ora = make_pair(rt, v, p)
    filler = [5] * 30 + [v.eos_id]
    for agent, arr, ert in ((0, 0, 220_000), (1, 1, 100_000_000), (2, 2, 100_000_000)):
        eng.submit(agent, [1], arr, ert, -2.0, 1.0, 0, 0, script=filler)
        ora.submit(agent, [1], arr, ert, -2.0, 1.0, 0, 0, script=filler)
    i = [eng.step() for _ in range(3)]
    assert [(x["t_us"], x["n_admitted"], x["n_refused_wcet"]) for x in i] == [(0, 1, 0), (21884, 1, 0), (44856, 0, 1)]
    for _ in range(3):
        ora.step()
    n, segs = lockstep(eng, ora)
    assert [s["dispatch_us"] for s in segs if s["request_id"] == 0][0] == 227720
