"""Agent timeline simulation and metrics (oracle c5, c10; test infrastructure only).

Waiting time of a segment: "the time between the completion of the preceding
segment's action, or the reception of the request in the case of the very
first segment, and the start of its own action" (fig:llm_time
PAPER.md:281).  Response time W(s_0); robot waiting time sum_k W(s_k); task
completion C(r) = sum_k (W(s_k) + E(s_k)).  Time utility =
TUF_0 at the actual response time.

c5: action_start_k = max(dispatch_k + net, action_end_{k-1})  (fig:con_infer
caption PAPER.md:217: network hidden when overlapped; 8 ms).
Realized duration of a skill = choice from its profiled alternatives by
splitmix64(seed ^ (request_id << 32) ^ ordinal) mod n, ordinal = the skill's index in the
request's whole response ("randomly sample from this profiled data"; reading
AMB-18) — independent of where segment boundaries fall, so the same trace served by
different systems executes the same actions.
"""
from .tuf import tuf0
from .weights import splitmix64_int, M64


def realized_us(vocab, seed, request_id, ordinal, tok):
    alts = vocab.realized[tok]
    h = splitmix64_int((seed ^ (request_id << 32) ^ ordinal) & M64)
    return int(alts[h % len(alts)])


def simulate_request(segments, arrival_us, vocab, net_us, seed, request_id):
    """segments: this request's records in k order -> per-segment (start, end, W, E)."""
    out = []
    prev_end = None
    ordinal = 0
    for s in sorted(segments, key=lambda s: s["k"]):
        E = 0
        for tok in s["tokens"]:
            if vocab.tok_skill[tok] >= 0:
                E += realized_us(vocab, seed, request_id, ordinal, tok)
                ordinal += 1
        start = s["dispatch_us"] + net_us
        if prev_end is not None:
            start = max(start, prev_end)
        W = start - (arrival_us if prev_end is None else prev_end)
        end = start + E
        out.append(dict(k=s["k"], start=start, end=end, W=W, E=E))
        prev_end = end
    return out


def request_metrics(segments, req, vocab, net_us, seed):
    tl = simulate_request(segments, req["arrival_us"], vocab, net_us, seed, req["request_id"])
    resp = tl[0]["W"]
    wait = sum(x["W"] for x in tl)
    comp = tl[-1]["end"] - req["arrival_us"]
    util = tuf0(req["beta"], req["alpha"], req["ert_us"], resp)
    return dict(request_id=req["request_id"], cls=req.get("cls"), response_us=resp, waiting_us=wait,
                completion_us=comp, exec_us=sum(x["E"] for x in tl), utility=util, timeline=tl)


def aggregate(metrics):
    """Per-class means ("averaged based on the task type")."""
    by = {}
    for m in metrics:
        by.setdefault(m["cls"], []).append(m)
    out = {}
    for c, ms in sorted(by.items(), key=lambda kv: str(kv[0])):
        n = len(ms)
        out[c] = dict(n=n, utility=sum(m["utility"] for m in ms) / n,
                      response_s=sum(m["response_us"] for m in ms) / n / 1e6,
                      waiting_s=sum(m["waiting_us"] for m in ms) / n / 1e6)
    return out
