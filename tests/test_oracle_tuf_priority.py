"""Pins for oracle c6 (TUF) and c7 (Eq. 4 priority).

P1/P2: values fixed by the paper's TUF presets and cut-offs and
SPEC.md:50-62 worked examples.  P3: closed forms of Eq. 4.
"""
import math
import random

import pytest

from oracle.tuf import tuf0, tuf1
from oracle.priority import priority, priority_seconds

S = 1_000_000


@pytest.mark.parametrize("t,expect", [(0.5, 1.0), (1.0, 1.0), (1.25, 0.5), (1.5, 0.0), (2.0, -1.0)])
def test_p1_normal(t, expect):
    # normal: ERT 1 s, beta 1, alpha -2; "cut-off time of 1.5 seconds"
    assert tuf0(1.0, -2.0, 1 * S, int(t * S)) == pytest.approx(expect, abs=1e-12)


@pytest.mark.parametrize("t,expect", [(0.2, 2.0), (0.35, 0.9995), (0.5, -0.001)])
def test_p1_urgent(t, expect):
    # urgent: ERT 200 ms, beta 2, alpha -6.67 "cut-off time of 0.5 s" (AMB-20)
    assert tuf0(2.0, -6.67, 200000, int(round(t * S))) == pytest.approx(expect, abs=1e-9)
    assert abs(tuf0(2.0, -6.67, 200000, 500000)) < 0.01


@pytest.mark.parametrize("t,expect", [(-3.0, 1.0), (0.0, 1.0), (0.25, 0.5)])
def test_p2_tuf1(t, expect):
    assert tuf1(1.0, -2.0, int(t * S)) == pytest.approx(expect, abs=1e-12)


def test_tuf_monotone_and_bounded():
    rng = random.Random(0)
    for _ in range(2000):
        beta = rng.uniform(-3, 3)
        alpha = -rng.uniform(0, 10)
        ert = rng.randint(0, 2 * S)
        a, b = sorted(rng.randint(-3 * S, 5 * S) for _ in range(2))
        assert tuf0(beta, alpha, ert, a) >= tuf0(beta, alpha, ert, b)
        assert tuf0(beta, alpha, ert, a) <= beta
        assert (tuf0(beta, alpha, ert, a) == beta) == (a <= ert or alpha == 0.0)
        # TUF1 == Eq.1 with ERT = 0 at max(t, 0)
        assert tuf1(beta, alpha, a) == tuf0(beta, alpha, 0, max(a, 0))


def test_p3_priority_worked_example():
    # k=0, TUF=1 (pre-deadline), G=0.09 s, L=0.86 s -> 12.92
    t = 0
    D = t + 90000 + 860000            # L = D - t - G = 0.86 s
    p = priority(t, 0, 0, D, D, -2.0, 1.0, 90000, 8000, 1000)
    assert p == pytest.approx(1.0 / (0.09 * 0.86), rel=1e-15)
    assert round(p, 4) == 12.9199


def test_p3_beta_ratio_exactly_two():
    # SPEC.md:287 / SPEC.md:342 scale invariance: beta and alpha scaled by 2
    for t in range(0, 900000, 37000):
        p1 = priority(t, 0, 0, 1 * S, 1 * S, -2.0, 1.0, 90000, 8000, 1000)
        p2 = priority(t, 0, 0, 1 * S, 1 * S, -4.0, 2.0, 90000, 8000, 1000)
        assert p2 == 2.0 * p1


def test_p3_fcfs_reduction():
    # two normal tasks arriving at 0.0 and 0.1, scored at t=0.2
    a = priority(200000, 0, 0, 1 * S, 1 * S, -2.0, 1.0, 90000, 8000, 1000)
    b = priority(200000, 0, 100000, 1100000, 1 * S, -2.0, 1.0, 90000, 8000, 1000)
    assert round(a, 4) == 15.6495 and round(b, 4) == 13.7174
    assert a > b


def test_p3_urgent_preempts_normal():
    # urgent arriving at 0.1 vs normal at 0.0, scored at t=0.1 (cf. Task 71/72)
    u = priority(100000, 0, 100000, 300000, 200000, -6.67, 2.0, 90000, 8000, 1000)
    n = priority(100000, 0, 0, 1 * S, 1 * S, -2.0, 1.0, 90000, 8000, 1000)
    assert round(u, 2) == 202.02 and round(n, 2) == 13.72


def test_pud_equals_fcfs_condition():
    # same class, k=0, t + G + net <= arrival + ERT for all -> priority decreasing in arrival
    rng = random.Random(1)
    for _ in range(200):
        t = rng.randint(0, 500000)
        arr = sorted(rng.randint(0, t) for _ in range(5))
        arr = [x for x in arr if t + 98000 <= x + S]
        pri = [priority(t, 0, x, x + S, S, -2.0, 1.0, 90000, 8000, 1000) for x in arr]
        assert all(pri[i] > pri[i + 1] for i in range(len(pri) - 1) if arr[i] < arr[i + 1])


def test_expired_slack_reading_amb3():
    # AMB-3: L floored at eps_L = 1 ms; just-expired with TUF > 0 dominates, negative sinks.
    t = 1_000_000
    p_exp = priority(t, 0, 0, S, S, -2.0, 1.0, 90000, 8000, 1000)   # W = 1.098 s, TUF 0.804
    assert p_exp == pytest.approx(0.804 / (0.09 * 0.001), rel=1e-12)
    p_neg = priority(1_500_000, 0, 0, S, S, -2.0, 1.0, 90000, 8000, 1000)  # W = 1.598 -> -0.196
    assert p_neg < 0


def test_negative_zero_canonical():
    # beta 0.0 pre-deadline -> num = 0.0; alpha*x + beta could give -0.0 for beta = -0.0
    p = priority(0, 0, 0, S, S, -2.0, -0.0, 90000, 8000, 1000)
    assert p == 0.0 and math.copysign(1.0, p) == 1.0


def test_suspended_priority_closed_form():
    # k>0: W = t + G + net - end_est; negative -> TUF1 = beta; L = end_est - t - G
    t, end = 1_000_000, 3_000_000
    p = priority(t, 1, end, end, S, -2.0, 1.0, 90000, 8000, 1000)
    assert p == pytest.approx(1.0 / (0.09 * 1.91), rel=1e-14)
    assert p == pytest.approx(priority_seconds(1.0, 1, 0.0, 3.0, 1.0, -2.0, 1.0, 0.09, 0.008,
                                               0.001, prev_end=3.0), rel=1e-12)
