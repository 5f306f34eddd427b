"""Segmented-generation round loop (oracle c2, c3, c4, c8, c9; test infrastructure only).

Follows the paper's serving loop step by step:
  * priority queue of initial + suspended generations; "evaluates resource
    availability whenever the LLM inference engine completes a decoding
    iteration, and when resources permit, it removes the highest-priority
    generation"  (§3)
  * all queued priorities are recomputed before fetching
  * WCET gate on the most urgent running generation + memory check, "a lag for
    one generation" (§4.4)
  * content-aware stop checker: suspend when executable skill(s) appear and
    dispatch the segment
  * context switching: KV pages + token ids retained, no re-prefill
    (§4.1)
  * suspended generations re-enter the queue with TUF_1 and the estimated
    completion of the previous segment

Exact round order (reading R-ROUND):
  1 ingest arrivals <= t          2 score all waiting (Eq. 4 or FCFS/EDF key)
  3 admit (key order; slot, memory, WCET, per-round cap)
  4 pop pages: k=0 admissions (prompt pages, admission order), then every
    decode slot (slot order) whose ctx % page == 0
  5 forward: k=0 admissions prefill and emit token 0; every other slot feeds
    its pending token and emits one token
  6 stop check (a9)   7 retire: suspend or finish + free   8 advance clock
"""
import math
import re

from .priority import priority
from . import model as M

STOP_NONE, STOP_EOS, STOP_MAXNEW, STOP_SKILL, STOP_CAP = 0, 1, 2, 3, 4
# Segmentation modes (the paper's comparison systems, PAPER.md:576-584,
# 657-661): SUSPEND = the method (segment ends, request suspended and re-queued,
# PAPER.md:180); STREAM = "vLLM-stream" (a segment is delivered at each skill boundary but
# the generation continues uninterrupted); NONE = "vLLM" (whole response delivered at the
# end).  Delivered segments are cut at SEG_MAX_TOKENS in STREAM / NONE.
SEG_SUSPEND, SEG_STREAM, SEG_NONE = 0, 1, 2
SEG_MAX_TOKENS = 128

# Stop grammars.  The paper's checker "detokenizes token IDs as they are
# generated in order to check an executable skill has been generated"
# with "regular expression matching"; chatbots end segments at sentences or
# paragraphs and execute them as reading time at 300 words per minute.
# The oracle does exactly that on the token TEXTS: GRAMMAR_SKILL appends each token's text
# to the text since the last complete statement and searches  name(digits);  at its end;
# the chat grammars count word-bearing tokens and test the token text for . ! ? / \n\n.
GRAMMAR_TOKEN, GRAMMAR_SKILL, GRAMMAR_SENTENCE, GRAMMAR_PARAGRAPH = 0, 1, 2, 3

# KV eviction to host memory + restore ("context caching":
# a suspended generation's KV moves to host memory when GPU memory is insufficient and is
# copied back on resume, 9.50 ms instead of a 133.31 ms re-prefill).  Reading R-EVICT
# (DESIGN.md): when a candidate that needs memory (k = 0, or an evicted resume) does not
# fit, suspended holders that come LATER in this round's key order are evicted, lowest
# priority first, if evicting them (within the host pool) makes it fit; an evicted request
# releases its whole reservation, its own pages go to host pages (host free stack, pops
# 0, 1, 2, ...), and it needs its reservation again to resume (memory check like k = 0),
# when it re-pops device pages in admission order and its KV is restored.
PENDING, WAITING, RUNNING, FINISHED = 0, 1, 2, 3
POLICY_PUD, POLICY_FCFS, POLICY_EDF = 0, 1, 2
CLOCK_VIRTUAL, CLOCK_WALL = 0, 1


class OracleError(ValueError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code  # "INVAL" | "NOMEM"


class OReq:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def ceil_div(a, b):
    return -(-a // b)


def wcet_gate_pass(max_seg_tokens, seg_tok, hist_sum_us, n, budget_us):
    """WCET = (max segment tokens - generated) / recent speed,
    speed = n tokens per hist_sum_us (mean of the last n round latencies, AMB-7).
    Pass iff WCET <= remaining budget, in exact integers:
    max(0, max_seg - seg_tok) * hist_sum <= n * budget."""
    if n <= 0:
        return True
    return max(0, max_seg_tokens - seg_tok) * hist_sum_us <= n * budget_us


class OracleEngine:
    def __init__(self, params, tok_skill, tok_exec_min_us, eos_id, vocab, model=None,
                 rank=0, world=1, grammar=None):
        self.p = params
        self.grammar = grammar  # tok_text, names, skill_base_us, skill_unit_us (NEXT-4)
        if grammar is not None:
            alts = "|".join(re.escape(n) for n in sorted(grammar.names, key=len, reverse=True))
            self._stmt_re = re.compile(r"(?<![A-Za-z])(" + alts + r")\((\d*)\);$")
            self._name_idx = {n: i for i, n in enumerate(grammar.names)}
        self.tok_skill = [int(x) for x in tok_skill]
        self.tok_e = [int(x) for x in tok_exec_min_us]
        self.eos = int(eos_id)
        self.vocab = int(vocab)
        self.model = model
        self.rank, self.world = rank, world
        self.t = int(params.t0_us)
        self.free = list(range(params.n_pages - 1, -1, -1))  # top = end; pops 0, 1, 2, ...
        self.host_pages = int(getattr(params, "host_pages", 0))
        self.hfree = list(range(self.host_pages - 1, -1, -1))  # host KV pages (R-EVICT)
        self.reqs = {}
        self.n_submitted = 0
        self.slots = []
        self.hist = []
        self.last_t = None
        self.last_nonempty = False
        self.segments = []
        self.round_log = []
        self.prefixes = []  # registered shared prefixes: dict(tokens, pages) (reading R-PFX)

    # ------------------------------------------------------------------ API
    def submit(self, agent_id, prompt, arrival_us, ert_us, alpha, beta, exec_window_us,
               max_new_tokens, script=None):
        p = self.p
        prompt = [int(x) for x in prompt]
        if not (alpha <= 0.0) or ert_us < 0 or not math.isfinite(beta) or exec_window_us < 0:
            raise OracleError("INVAL", "bad utility function")
        if agent_id < 0:
            raise OracleError("INVAL", "bad agent")
        if len(prompt) < 1 or any(t < 0 or t >= self.vocab for t in prompt):
            raise OracleError("INVAL", "bad prompt")
        if script is not None:
            script = [int(x) for x in script]
            if len(script) < 1 or any(t < 0 or t >= self.vocab for t in script):
                raise OracleError("INVAL", "bad script")
            max_new_tokens = len(script)
        if max_new_tokens < 1 or len(prompt) + max_new_tokens > p.max_ctx:
            raise OracleError("INVAL", "context too long")
        R = ceil_div(len(prompt) + max_new_tokens, p.page_tokens)
        pfx, npfx = self._match_prefix(prompt)
        if R - npfx > p.n_pages:
            raise OracleError("NOMEM", "request larger than pool")
        live = sum(1 for r in self.reqs.values() if not r.polled_final)
        if live >= p.max_tasks:
            raise OracleError("NOMEM", "task table full")
        rid = self.n_submitted * self.world + self.rank
        self.n_submitted += 1
        self.reqs[rid] = OReq(
            id=rid, agent=int(agent_id), arrival=int(arrival_us), ert=int(ert_us),
            alpha=float(alpha), beta=float(beta), window=int(exec_window_us),
            prompt=prompt, script=script, max_new=int(max_new_tokens), state=PENDING,
            k=0, D=int(arrival_us) + int(ert_us), ref=int(arrival_us), end_est=None,
            n_gen=0, seg_tok=0, seg_exec=0, seg_nsk=0, pending=None, ctx=0, pages=[],
            R=R, holder=False, out=[], polled_final=False, argmax=[], pfx=pfx, npfx=npfx,
            evicted=False, hpages=[], stmt_text="")
        return rid

    def register_prefix(self, tokens):
        """Shared prompt prefix (PAPER.md:211 fixed prompt components stored
        on the server; DESIGN R-PFX): len a positive multiple of page_tokens below max_ctx.
        Pops len/16 pages now (admission pop order), keeps them read-only forever, and
        computes their KV once."""
        p = self.p
        tokens = [int(x) for x in tokens]
        n = len(tokens) // p.page_tokens
        if (len(tokens) < p.page_tokens or len(tokens) % p.page_tokens or len(tokens) >= p.max_ctx
                or any(t < 0 or t >= self.vocab for t in tokens)):
            raise OracleError("INVAL", "bad prefix")
        if len(self.prefixes) >= 8:
            raise OracleError("NOMEM", "too many prefixes")
        if self._avail() < n:
            raise OracleError("NOMEM", "not enough free pages for the prefix")
        pages = [self.free.pop() for _ in range(n)]
        pid = len(self.prefixes)
        self.prefixes.append(dict(tokens=tokens, pages=pages))
        if self.model is not None:
            self.model.forward([(("pfx", pid), i, t) for i, t in enumerate(tokens)])
        return pid

    def _match_prefix(self, prompt):
        """Longest registered prefix that is a proper head of the prompt -> (id, pages)."""
        best, npfx = -1, 0
        for i, pf in enumerate(self.prefixes):
            lp = len(pf["tokens"])
            if lp < len(prompt) and lp // self.p.page_tokens > npfx and prompt[:lp] == pf["tokens"]:
                best, npfx = i, lp // self.p.page_tokens
        return best, npfx

    def poll(self):
        out, self.segments = self.segments, []
        for s in out:
            if s["reason"] in (STOP_EOS, STOP_MAXNEW):
                self.reqs[s["request_id"]].polled_final = True
        return out

    def page_tables(self):
        return {r.id: list(r.pages) for r in self.reqs.values() if r.holder}

    def host_page_tables(self):
        return {r.id: list(r.hpages) for r in self.reqs.values() if r.evicted}

    # ---------------------------------------------------------------- round
    def _ingest(self, t):
        for rid in sorted(self.reqs):
            r = self.reqs[rid]
            if r.state == PENDING and r.arrival <= t:
                r.state = WAITING

    def _key(self, r, t):
        p = self.p
        if p.policy == POLICY_PUD:
            r.pri = priority(t, r.k, r.ref, r.D, r.ert, r.alpha, r.beta, p.g_us, p.net_us, p.eps_l_us)
            return (-r.pri, r.arrival, r.id)
        if p.policy == POLICY_FCFS:
            return (r.arrival, r.id)
        return (r.arrival + r.ert, r.arrival, r.id)  # EDF on the initial deadline

    def _avail(self):
        return len(self.free) - sum(r.R - len(r.pages) for r in self.reqs.values() if r.holder)

    def step(self, now_us=None):
        p = self.p
        if p.clock_mode == CLOCK_WALL:
            t = int(now_us)
            if self.last_nonempty:
                self.hist.append(t - self.last_t)
            self.last_nonempty = False
            self.last_t = t
        else:
            t = self.t
        self._ingest(t)
        running = [self.reqs[i] for i in self.slots]
        waiting = [r for r in self.reqs.values() if r.state == WAITING]
        if not running and not waiting:
            pend = [r.arrival for r in self.reqs.values() if r.state == PENDING]
            if p.clock_mode == CLOCK_VIRTUAL and pend:
                t = min(pend)
                self.t = t
                self._ingest(t)
                waiting = [r for r in self.reqs.values() if r.state == WAITING]
            else:
                info = dict(t_us=t, round_us=0, n_waiting=0, n_running=0, n_admitted=0,
                            n_stopped=0, n_refused_mem=0, n_refused_wcet=0)
                return info
        n_waiting = len(waiting)
        order = sorted(waiting, key=lambda r: self._key(r, t))
        # local top-K candidates {Pri (0 for FCFS/EDF), arrival, id, rank} (c13 / a12)
        topk = [((r.pri if p.policy == POLICY_PUD else 0.0), r.arrival, r.id, self.rank)
                for r in order[:16]]

        # ---- WCET gate, judged on history up to round r-1 (AMB-8)
        n = min(p.speed_window, len(self.hist))
        S = sum(self.hist[len(self.hist) - n:]) if n else 0
        gate_ok = True
        cands = [g for g in running if g.D - t >= 0]
        if cands and n > 0 and not getattr(p, "wcet_off", 0):
            g = min(cands, key=lambda g: (g.D - t, g.id))
            gate_ok = wcet_gate_pass(p.max_seg_tokens, g.seg_tok, S, n, g.D - t)

        # ---- admission (c8 + reading R-MEM; eviction R-EVICT)
        admitted = []
        evicted_now = []
        refused_mem = refused_wcet = 0
        mem_blocked = False
        avail = self._avail()
        havail = len(self.hfree)
        for ci, c in enumerate(order):
            if len(admitted) >= p.max_admit_per_round:
                break
            if len(running) + len(admitted) >= p.max_batch:
                break
            if not gate_ok:
                refused_wcet = 1
                break
            if c in evicted_now:          # evicted earlier in this round: not resumable now
                refused_mem += 1
                continue
            if c.k == 0 or c.evicted:  # own pages only: a shared prefix is already resident (R-PFX)
                need = c.R - c.npfx
                if not mem_blocked and avail < need and self.host_pages > 0:
                    # victims: suspended holders later in the key order, lowest priority first
                    vict, gain, hneed = [], 0, 0
                    for v in reversed(order[ci + 1:]):
                        if avail + gain >= need:
                            break
                        if v.k > 0 and v.holder and not v.evicted and v not in evicted_now:
                            own = len(v.pages) - v.npfx
                            if hneed + own > havail:
                                continue
                            vict.append(v)
                            gain += v.R - v.npfx
                            hneed += own
                    if avail + gain >= need:
                        for v in vict:
                            evicted_now.append(v)
                            avail += v.R - v.npfx
                            havail -= len(v.pages) - v.npfx
                if mem_blocked or avail < need:
                    mem_blocked = True
                    refused_mem += 1
                    continue
                avail -= need
            admitted.append(c)

        # ---- evictions: own pages -> host pages, device pages pushed back (R-EVICT)
        swaps = []  # (direction, rid, device page, host page); 0 = to host, 1 = restore
        for v in evicted_now:
            own = v.pages[v.npfx:]
            v.hpages = [self.hfree.pop() for _ in own]
            swaps += [(0, v.id, dp, hp) for dp, hp in zip(own, v.hpages)]
            for pg in reversed(own):
                self.free.append(pg)
            v.pages = v.pages[:v.npfx]
            v.holder = False
            v.evicted = True

        # ---- page allocation + batch assembly (c2, AMB-14)
        popped = []
        prefill = set()
        restored = []
        for a in admitted:
            a.state = RUNNING
            if a.k == 0:
                prefill.add(a.id)
                a.holder = True
                if a.pfx >= 0:
                    a.pages = list(self.prefixes[a.pfx]["pages"])
                for _ in range(ceil_div(len(a.prompt), p.page_tokens) - a.npfx):
                    pg = self.free.pop()
                    a.pages.append(pg)
                    popped.append((a.id, pg))
            elif a.evicted:  # restore: re-pop its own pages, KV copied back from host
                a.holder = True
                a.evicted = False
                for hp in a.hpages:
                    pg = self.free.pop()
                    a.pages.append(pg)
                    popped.append((a.id, pg))
                    swaps.append((1, a.id, pg, hp))
                restored.append(a)
        for a in restored:  # host pages back (reverse order), in admission order
            for hp in reversed(a.hpages):
                self.hfree.append(hp)
            a.hpages = []
        slots = self.slots + [a.id for a in admitted]
        for rid in slots:
            r = self.reqs[rid]
            if rid in prefill:
                continue
            if r.ctx % p.page_tokens == 0:
                pg = self.free.pop()
                r.pages.append(pg)
                popped.append((rid, pg))

        # ---- forward (rows) + token selection (c3)
        rows, last_row = [], {}
        sum_ctx = sum_prompt = 0
        for rid in slots:
            r = self.reqs[rid]
            if rid in prefill:
                lp = r.npfx * p.page_tokens  # prefix positions are not recomputed (R-PFX)
                if r.pfx >= 0 and self.model is not None:
                    self.model.share_prefix(("pfx", r.pfx), rid, lp)
                for i in range(lp, len(r.prompt)):
                    rows.append((rid, i, r.prompt[i]))
                last_row[rid] = len(rows) - 1
                r.ctx = len(r.prompt)
                sum_prompt += len(r.prompt) - lp
            else:
                rows.append((rid, r.ctx, r.pending))
                last_row[rid] = len(rows) - 1
                r.ctx += 1
                sum_ctx += r.ctx
        argmax = {}
        logits = {}
        if self.model is not None:
            hid = self.model.forward(rows)
            for rid in slots:
                lg = self.model.logits(hid[last_row[rid]][None, :])[0]
                logits[rid] = lg
                argmax[rid] = M.argmax_lowest(lg)

        B = len(slots)
        if p.clock_mode == CLOCK_VIRTUAL:
            round_us = (p.base_us + (p.base_us * p.gamma_ppm * (B - 1)) // 1000000
                        + (p.kv_us_per_1k * sum_ctx) // 1024 + p.prefill_us_per_tok * sum_prompt
                        + getattr(p, "swap_us_per_page", 0) * len(swaps))
            dispatch = t + round_us
        else:
            round_us = self.hist[-1] if self.hist else 0
            dispatch = t + round_us

        # ---- stop checker (c4 / a9) per slot in slot order
        stops, toks = [], []
        for rid in slots:
            r = self.reqs[rid]
            if r.script is not None:
                tok = r.script[r.n_gen]
            else:
                tok = argmax[rid]
            r.argmax.append(argmax.get(rid))
            toks.append(tok)
            r.n_gen += 1
            r.seg_tok += 1
            r.out.append(tok)
            r.pending = tok
            sk = self._stop_unit(r, tok)
            if sk >= 0:
                r.seg_nsk += 1
            mode = getattr(p, "seg_mode", SEG_SUSPEND)
            cap = p.max_seg_tokens if mode == SEG_SUSPEND else SEG_MAX_TOKENS
            if tok == self.eos:
                reason = STOP_EOS
            elif r.n_gen == r.max_new:
                reason = STOP_MAXNEW
            elif mode != SEG_NONE and sk >= 0 and r.seg_exec >= r.window:
                reason = STOP_SKILL
            elif r.seg_tok == cap:
                reason = STOP_CAP
            else:
                reason = STOP_NONE
            if reason != STOP_NONE:
                stops.append((rid, reason))

        # ---- retire (a10)
        finished = []
        stopped_ids = set()
        for rid, reason in stops:
            r = self.reqs[rid]
            stopped_ids.add(rid)
            self.segments.append(dict(
                request_id=rid, agent_id=r.agent, k=r.k, tok_begin=r.n_gen - r.seg_tok,
                tok_end=r.n_gen, n_skills=r.seg_nsk, est_exec_us=r.seg_exec, reason=reason,
                dispatch_us=dispatch, tokens=list(r.out[r.n_gen - r.seg_tok:r.n_gen])))
            if reason in (STOP_EOS, STOP_MAXNEW):
                finished.append(r)
            elif getattr(p, "seg_mode", SEG_SUSPEND) != SEG_SUSPEND:
                # STREAM / NONE cut: delivered, the generation goes on in its slot
                r.k += 1
                r.seg_tok = r.seg_exec = r.seg_nsk = 0
                stopped_ids.discard(rid)
            else:
                base = dispatch + p.net_us
                if r.end_est is not None:
                    base = max(base, r.end_est)
                r.end_est = base + r.seg_exec
                r.D = r.end_est
                r.ref = r.end_est
                r.k += 1
                r.seg_tok = r.seg_exec = r.seg_nsk = 0
                r.state = WAITING
        for r in sorted(finished, key=lambda r: r.id):
            for pg in reversed(r.pages[r.npfx:]):  # own pages; the prefix's stay (R-PFX)
                self.free.append(pg)
            r.pages = []
            r.holder = False
            r.state = FINISHED
            if self.model is not None:
                self.model.drop(r.id)
        self.slots = [rid for rid in slots if rid not in stopped_ids]

        if p.clock_mode == CLOCK_VIRTUAL:
            self.t = t + round_us
            self.hist.append(round_us)
        else:
            self.last_nonempty = True

        info = dict(t_us=t, round_us=round_us, n_waiting=n_waiting, n_running=B,
                    n_admitted=len(admitted), n_stopped=len(stops), n_refused_mem=refused_mem,
                    n_refused_wcet=refused_wcet, n_evicted=len(evicted_now), n_restored=len(restored))
        self.round_log.append(dict(info, admitted=[a.id for a in admitted], slots=list(slots), swaps=swaps,
                                   tokens=toks, argmax=[argmax.get(r) for r in slots],
                                   stops=stops, popped=popped, free=len(self.free), topk=topk,
                                   logits=logits if self.model is not None else None))
        return info

    # -------------------------------------------------------------- helpers
    def _stop_unit(self, r, tok):
        """Does token `tok` complete an executable unit of request r (>= 0) — and add its
        execution estimate to the segment (c4 / a9, per stop grammar)."""
        g = getattr(self.p, "stop_grammar", GRAMMAR_TOKEN)
        if g == GRAMMAR_TOKEN:
            sk = self.tok_skill[tok]
            if sk >= 0:
                r.seg_exec += self.tok_e[tok]
            return sk
        text = self.grammar.tok_text[tok]
        if g == GRAMMAR_SKILL:
            r.stmt_text += text
            m = self._stmt_re.search(r.stmt_text)
            if m is None:
                return -1
            name = m.group(1)
            arg = min(int(m.group(2)) if m.group(2) else 0, 1000000)
            i = self._name_idx[name]
            r.seg_exec += int(self.grammar.skill_base_us[i]) + int(self.grammar.skill_unit_us[i]) * arg
            r.stmt_text = ""
            return i
        if re.search(r"[A-Za-z0-9]", text):      # a word (reading time, 300 wpm)
            r.seg_exec += int(getattr(self.p, "word_us", 200000))
        if text == "\n\n" or (g == GRAMMAR_SENTENCE and text in (".", "!", "?")):
            return 0
        return -1

    def run_until_idle(self, max_rounds=100000):
        for _ in range(max_rounds):
            info = self.step()
            if info["n_running"] == 0 and not any(
                    r.state in (PENDING, WAITING) for r in self.reqs.values()):
                return
        raise RuntimeError("not quiescent")
