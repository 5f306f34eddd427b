"""Host-side time-utility report of a segment log (not on the device hot path).

Definitions (fig:llm_time PAPER.md:281, metrics PAPER.md:586-593):
response time W(s_0) = first action start - arrival; robot waiting time
sum_k W(s_k); completion C = sum_k (W(s_k) + E(s_k)); time utility = Eq. 1 at
the response time.  Agents are simulated in virtual time: action k starts at
max(dispatch_k + net, end of action k-1) (fig:con_infer) and lasts
the sum of its skills' realized durations, sampled per (request, skill ordinal in the
whole response) by splitmix64(seed ^ (rid << 32) ^ ordinal) — independent
of segment boundaries, so every serving mode (rt.h RT_SEG_*) executes the same actions.
"""
M64 = (1 << 64) - 1


def _mix(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def utility(beta, alpha, ert_us, w_us):
    y = beta + alpha * ((w_us - ert_us) / 1e6)
    return beta if beta <= y else y


def report(segments, requests, vocab, net_us=8000, seed=0, exec_from="tokens", per_request=False):
    """segments: rt_poll_segment records; requests: {rid: dict(arrival_us, beta, alpha,
    ert_us, cls)}.  Returns per-class means and totals over completed requests (and, with
    per_request, the per-request figures under "requests").
    exec_from="est": a segment executes for its est_exec_us (multi-token stop grammars, e.g.
    the chatbot's reading time) instead of sampled per-skill durations."""
    by_rid = {}
    for s in segments:
        by_rid.setdefault(s["request_id"], []).append(s)
    per = []
    for rid, segs in by_rid.items():
        req = requests.get(rid)
        if req is None or not any(s["reason"] in (1, 2) for s in segs):
            continue
        prev_end = None
        waits = []
        e_tot = 0
        ordinal = 0
        for s in sorted(segs, key=lambda s: s["k"]):
            e = s["est_exec_us"] if exec_from == "est" else 0
            for tok in (s["tokens"] if exec_from != "est" else ()):
                if vocab.tok_skill[tok] >= 0:
                    alts = vocab.realized[tok]
                    e += alts[_mix((seed ^ (rid << 32) ^ ordinal) & M64) % len(alts)]
                    ordinal += 1
            start = s["dispatch_us"] + net_us if prev_end is None else max(s["dispatch_us"] + net_us, prev_end)
            waits.append(start - (req["arrival_us"] if prev_end is None else prev_end))
            prev_end = start + e
            e_tot += e
        per.append(dict(request_id=rid, cls=req.get("cls"), response_us=waits[0], waiting_us=sum(waits),
                        completion_us=prev_end - req["arrival_us"], exec_us=e_tot,
                        utility=utility(req["beta"], req["alpha"], req["ert_us"], waits[0])))
    out = {}
    for m in per:
        out.setdefault(m["cls"], []).append(m)
    summary = {c: dict(n=len(v), utility=sum(m["utility"] for m in v) / len(v),
                       response_s=sum(m["response_us"] for m in v) / len(v) / 1e6,
                       waiting_s=sum(m["waiting_us"] for m in v) / len(v) / 1e6) for c, v in out.items()}
    total = sum(m["utility"] for m in per)
    n = len(per)
    out = dict(by_class=summary, n=n, total_utility=total,
               mean_utility=(total / n) if per else None,
               mean_response_s=(sum(m["response_us"] for m in per) / n / 1e6) if per else None,
               mean_waiting_s=(sum(m["waiting_us"] for m in per) / n / 1e6) if per else None)
    if per_request:
        out["requests"] = per
    return out
