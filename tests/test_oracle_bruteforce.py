"""Pins for oracle c12 (Eq. 3 brute force, Theorem 1) and c13 (global merge, P13)."""
import math
import random

import pytest

from oracle import bruteforce as BF
from oracle.merge import global_topk, merge_rank_topk

TICK = 10000  # 10 ms


def inst_random(rng, n_req, max_seg):
    inst = []
    for i in range(n_req):
        urgent = rng.random() < 0.4
        ns = rng.randint(1, max_seg)
        inst.append(dict(arrival=rng.randint(0, 4) * TICK,
                         g=[rng.randint(1, 4) * TICK for _ in range(ns)],
                         e=[rng.randint(1, 8) * TICK for _ in range(ns)],
                         beta=2.0 if urgent else 1.0, alpha=-6.67 if urgent else -2.0,
                         ert=(2 if urgent else 6) * TICK))
    return inst


def test_enumeration_counts():
    inst = [dict(arrival=0, g=[TICK] * a, e=[TICK] * a, beta=1.0, alpha=-1.0, ert=0)
            for a in (3, 3, 3)]
    assert len(BF.brute_force(inst)) == math.factorial(9) // 6 ** 3        # 1680
    inst2 = inst[:2]
    assert len(BF.brute_force(inst2)) == math.factorial(6) // 36            # 20
    one = [dict(arrival=0, g=[TICK], e=[TICK], beta=1.0, alpha=-1.0, ert=0)] * 2
    assert len(BF.brute_force(one)) == 2


def test_eq3_examples():
    # single request served immediately -> beta; second segment
    # generated before the first action ends -> 2 beta; late -> Eq. 1 arithmetic
    r = dict(arrival=0, g=[TICK], e=[5 * TICK], beta=1.0, alpha=-2.0, ert=2 * TICK)
    assert BF.evaluate([r], (0,))[0] == 1.0
    r2 = dict(arrival=0, g=[TICK, TICK], e=[5 * TICK, TICK], beta=1.0, alpha=-2.0, ert=2 * TICK)
    assert BF.evaluate([r2], (0, 0))[0] == 2.0
    r3 = dict(arrival=0, g=[50 * TICK], e=[TICK], beta=1.0, alpha=-2.0, ert=10 * TICK)
    assert BF.evaluate([r3], (0,))[0] == pytest.approx(1.0 - 2.0 * 0.4)


def test_p9_greedy_le_opt_and_equality_cases():
    rng = random.Random(11)
    for _ in range(60):
        inst = inst_random(rng, rng.randint(1, 3), 3)
        best, _, _ = BF.optimum(inst)
        g = BF.greedy_pud(inst, g_us=2 * TICK)
        gv = BF.evaluate(inst, g)[0]
        assert gv <= best + 1e-12
        if len(inst) == 1:
            assert gv == pytest.approx(best)
    # uncontended: ready times never overlap -> any work-conserving order is optimal
    inst = [dict(arrival=0, g=[TICK, TICK], e=[3 * TICK, TICK], beta=1.0, alpha=-2.0, ert=5 * TICK),
            dict(arrival=100 * TICK, g=[TICK], e=[TICK], beta=2.0, alpha=-6.67, ert=2 * TICK)]
    best, _, _ = BF.optimum(inst)
    assert BF.evaluate(inst, BF.greedy_pud(inst, g_us=TICK))[0] == pytest.approx(best)


def test_theorem1_counterexample_hand_worked():
    """FINDING (DESIGN.md F-THM1): Theorem 1 does not hold under the
    paper's own definitions.  Hand-worked (ms):
      U: arrival 30, g=[40,30,20], e=[50,20,30], beta 2, alpha -6.67, ERT 20
      N: arrival 40, g=[20,10,20], e=[30,50,80], beta 1, alpha -2,    ERT 60
      x* = (U0,U1,N0,U2,N1,N2): U W=[40,0,0] -> 1.8666+2+2; N W=[80,0,0] -> 0.96+1+1
           Eq.3 = 8.8266, C = (140, 240), TUF0 = (1.8666, 0.96)
      x' = (U0,N0,U1,U2,N1,N2): U W=[40,0,0];  N W=[50,30,0] -> 1+0.94+1
           Eq.3 = 8.8066, C = (140, 240), TUF0 = (1.8666, 1.0)
    x' Pareto-dominates the unique Eq. 3 optimum x* (same completions, higher
    first-segment utility): Lemma 3's "no other segment negatively impacted" fails
    (N's second segment waits 30 ms longer)."""
    ms = 1000
    inst = [dict(arrival=30 * ms, g=[40 * ms, 30 * ms, 20 * ms], e=[50 * ms, 20 * ms, 30 * ms],
                 beta=2.0, alpha=-6.67, ert=20 * ms),
            dict(arrival=40 * ms, g=[20 * ms, 10 * ms, 20 * ms], e=[30 * ms, 50 * ms, 80 * ms],
                 beta=1.0, alpha=-2.0, ert=60 * ms)]
    xs, xp = (0, 0, 1, 0, 1, 1), (0, 1, 0, 0, 1, 1)
    v1, C1, U1, W1 = BF.evaluate(inst, xs)
    v2, C2, U2, W2 = BF.evaluate(inst, xp)
    assert W1 == [[40 * ms, 0, 0], [80 * ms, 0, 0]] and W2 == [[40 * ms, 0, 0], [50 * ms, 30 * ms, 0]]
    assert v1 == pytest.approx(8.8266, abs=1e-12) and v2 == pytest.approx(8.8066, abs=1e-12)
    assert C1 == C2 == [140 * ms, 240 * ms]
    assert U1 == pytest.approx([1.8666, 0.96]) and U2 == pytest.approx([1.8666, 1.0])
    best, argmax, res = BF.optimum(inst)
    assert [a[0] for a in argmax] == [xs] and best == pytest.approx(v1)
    assert BF.dominates(C2, U2, C1, U1)
    assert (xs, xp) in BF.pareto_counterexamples(inst)


def test_eq3_decomposition_identity():
    # Eq.3 = sum_i [TUF0(W0) + |alpha| W0] - sum_i |alpha| (C - E) + sum_i K beta (exact algebra)
    rng = random.Random(7)
    for _ in range(40):
        inst = inst_random(rng, rng.randint(1, 3), 3)
        for od, obj, C, U in BF.brute_force(inst, work_conserving_only=False):
            assert BF.eq3_decomposition(inst, od) == pytest.approx(obj, abs=1e-9)


def test_lemma2_holds_at_fixed_first_segment_waits():
    """What does hold (DESIGN.md F-THM1): among schedules with the same first-segment
    waiting times, the Eq. 3 maximiser minimises sum |alpha_i| C_i and no schedule
    of the group Pareto-improves its completion times."""
    rng = random.Random(2024)
    for _ in range(150):
        inst = inst_random(rng, rng.randint(2, 3), 3)
        groups = {}
        for od in BF._orders([len(r["g"]) for r in inst]):
            obj, C, U, W = BF.evaluate(inst, od)
            groups.setdefault(tuple(w[0] for w in W), []).append((obj, C))
        for g in groups.values():
            best = max(o for o, _ in g)
            for o, C in g:
                if o >= best - 1e-12:
                    wc = sum(-r["alpha"] * c for r, c in zip(inst, C))
                    assert all(wc <= sum(-r["alpha"] * c2 for r, c2 in zip(inst, C2)) + 1e-6
                               for _, C2 in g)
                    assert not any(all(a <= b for a, b in zip(C2, C)) and C2 != C for _, C2 in g)


def test_p13_global_merge():
    rng = random.Random(5)
    for _ in range(200):
        G = rng.randint(1, 8)
        K = rng.randint(1, 16)
        per_rank = []
        union = []
        for rank in range(G):
            recs = []
            for j in range(rng.randint(0, 40)):
                pri = rng.choice([rng.uniform(-50, 300), 13.5, 0.0])   # ties exercised
                recs.append((pri, rng.randint(0, 10) * 1000, j * G + rank, rank))
            union += recs
            per_rank.append(global_topk(recs, K))
        assert merge_rank_topk(per_rank, K) == global_topk(union, K)
        assert merge_rank_topk(per_rank, K) == sorted(union, key=lambda r: (-r[0], r[1], r[2]))[:K]
