"""Brute-force Eq. 3 optimum and Theorem 1 check on tiny instances
(oracle c12; test infrastructure only).

Eq. 3:  max sum_i [ TUF_0^i(W(s_0^i)) + sum_{k>=1} TUF_1^i(W(s_k^i)) ]
Theorem 1 (Appendix A): with monotone
non-increasing TUFs, the Eq. 3 optimum is Pareto optimal w.r.t. the request
completion times C(r^i) and the first-segment utilities.

Instance model: one batch-1 generation server,
non-preemptive segment generations, segment k+1 of a request is generated after
segment k; the robot starts action k at max(generation end, end of action
k-1) (zero network here).  Schedule space = all precedence-respecting orders,
each generation started as early as possible (work-conserving, as the
paper's engine).  Times are integer microseconds.
"""
from .tuf import tuf0, tuf1
from .priority import priority


def _orders(counts):
    """All interleavings of requests with counts[i] segments (multiset permutations)."""
    n = sum(counts)
    rem = list(counts)
    seq = []

    def rec():
        if len(seq) == n:
            yield tuple(seq)
            return
        for i in range(len(rem)):
            if rem[i]:
                rem[i] -= 1
                seq.append(i)
                yield from rec()
                seq.pop()
                rem[i] += 1
    yield from rec()


def evaluate(inst, order):
    """inst: list of dict(arrival, g: [..], e: [..], beta, alpha, ert).  Returns
    (objective, C list, TUF0 list, W lists)."""
    free = 0
    nxt = [0] * len(inst)
    gen_end = [[None] * len(r["g"]) for r in inst]
    for i in order:
        r = inst[i]
        j = nxt[i]
        ready = r["arrival"] if j == 0 else gen_end[i][j - 1]
        start = max(free, ready)
        gen_end[i][j] = start + r["g"][j]
        free = gen_end[i][j]
        nxt[i] += 1
    obj = 0.0
    Cs, U0, Ws = [], [], []
    for i, r in enumerate(inst):
        prev_end = None
        W = []
        for j in range(len(r["g"])):
            st = gen_end[i][j] if prev_end is None else max(gen_end[i][j], prev_end)
            W.append(st - (r["arrival"] if prev_end is None else prev_end))
            prev_end = st + r["e"][j]
        u0 = tuf0(r["beta"], r["alpha"], r["ert"], W[0])
        obj += u0 + sum(tuf1(r["beta"], r["alpha"], w) for w in W[1:])
        Cs.append(prev_end - r["arrival"])
        U0.append(u0)
        Ws.append(W)
    return obj, Cs, U0, Ws


def work_conserving(inst, order):
    """True iff the server never idles while another segment is ready: whenever
    the next segment in ``order`` is not ready when the server frees up, no
    other eligible segment may become ready earlier than it."""
    free = 0
    nxt = [0] * len(inst)
    gen_end = [[None] * len(r["g"]) for r in inst]

    def ready(q):
        return inst[q]["arrival"] if nxt[q] == 0 else gen_end[q][nxt[q] - 1]
    for i in order:
        r_i = ready(i)
        if r_i > free:
            for q in range(len(inst)):
                if q != i and nxt[q] < len(inst[q]["g"]) and ready(q) < r_i:
                    return False
        j = nxt[i]
        gen_end[i][j] = max(free, r_i) + inst[i]["g"][j]
        free = gen_end[i][j]
        nxt[i] += 1
    return True


def brute_force(inst, work_conserving_only=True):
    """Every precedence-respecting order (optionally only work-conserving ones):
    list of (order, obj, C, U0)."""
    res = []
    for od in _orders([len(r["g"]) for r in inst]):
        if work_conserving_only and not work_conserving(inst, od):
            continue
        obj, C, U0, _ = evaluate(inst, od)
        res.append((od, obj, C, U0))
    return res


def optimum(inst, tol=1e-12, work_conserving_only=True):
    res = brute_force(inst, work_conserving_only)
    best = max(r[1] for r in res)
    return best, [r for r in res if r[1] >= best - tol], res


def dominates(C2, U2, C, U, tol=1e-12):
    le = all(c2 <= c for c2, c in zip(C2, C)) and all(u2 >= u - tol for u2, u in zip(U2, U))
    strict = any(c2 < c for c2, c in zip(C2, C)) or any(u2 > u + tol for u2, u in zip(U2, U))
    return le and strict


def pareto_counterexamples(inst, tol=1e-12, work_conserving_only=True):
    """Schedules that Pareto-dominate an Eq. 3 argmax in (C_i <=, TUF0_i >=, one strict)."""
    best, argmax, res = optimum(inst, tol, work_conserving_only)
    bad = []
    for (od, _, C, U) in argmax:
        for (od2, _, C2, U2) in res:
            if dominates(C2, U2, C, U, tol):
                bad.append((od, od2))
    return bad


def eq3_decomposition(inst, order):
    """Exact algebra of Eq. 3 under this model (W_k >= 0 for k >= 1, so TUF_1 is
    linear): sum_i [TUF_0(W_0) + |alpha| W_0] - sum_i |alpha| (C_i - E_i) + sum_i K_i beta."""
    _, C, U0, Ws = evaluate(inst, order)
    tot = 0.0
    for r, c, u0, W in zip(inst, C, U0, Ws):
        a = -r["alpha"]
        E = sum(r["e"])
        tot += u0 + a * W[0] / 1e6 - a * (c - E) / 1e6 + (len(r["g"]) - 1) * r["beta"]
    return tot


def greedy_pud(inst, g_us, net_us=0, eps_l_us=1000):
    """The paper's greedy at batch 1: at every scheduling point pick
    the ready segment with the highest Eq. 4 priority (ties: arrival, index)."""
    n = len(inst)
    nxt = [0] * n
    gen_end = [[None] * len(r["g"]) for r in inst]
    end_est = [None] * n
    t = 0
    order = []
    total = sum(len(r["g"]) for r in inst)
    while len(order) < total:
        ready = []
        for i, r in enumerate(inst):
            j = nxt[i]
            if j >= len(r["g"]):
                continue
            rt = r["arrival"] if j == 0 else gen_end[i][j - 1]
            if rt <= t:
                ready.append(i)
        if not ready:
            t = min((inst[i]["arrival"] if nxt[i] == 0 else gen_end[i][nxt[i] - 1])
                    for i in range(n) if nxt[i] < len(inst[i]["g"]))
            continue

        def key(i):
            r = inst[i]
            j = nxt[i]
            ref = r["arrival"] if j == 0 else end_est[i]
            D = r["arrival"] + r["ert"] if j == 0 else end_est[i]
            pri = priority(t, j, ref, D, r["ert"], r["alpha"], r["beta"], g_us, net_us, eps_l_us)
            return (-pri, r["arrival"], i)
        i = min(ready, key=key)
        j = nxt[i]
        gen_end[i][j] = t + inst[i]["g"][j]
        disp = gen_end[i][j]
        base = disp + net_us if end_est[i] is None else max(disp + net_us, end_est[i])
        end_est[i] = base + inst[i]["e"][j]
        t = gen_end[i][j]
        nxt[i] += 1
        order.append(i)
    return tuple(order)
