"""Eq. 1 and TUF1 (oracle, test infrastructure only).

PAPER.md:136-139 (§2.3, Eq. 1):   TUF(t) = min(beta, alpha * (t - ERT) + beta)
PAPER.md:271-272 (§4.2):          TUF_1(t) = min(beta, alpha * max(t, 0) + beta)

Times enter as integer microseconds (reading AMB-23); seconds appear only as
one correctly-rounded division x_us / 1e6.  Operation order (fixed, no FMA):
x = float(int) / 1e6 ; y = alpha * x ; y = y + beta ; min(beta, y).
"""


def tuf0(beta: float, alpha: float, ert_us: int, w_us: int) -> float:
    """Eq. 1 evaluated at waiting / response time w_us (µs)."""
    x = float(int(w_us) - int(ert_us)) / 1e6
    y = alpha * x
    y = y + beta
    return beta if beta <= y else y


def tuf1(beta: float, alpha: float, w_us: int) -> float:
    """TUF_1 of a suspended generation: ERT := 0, negative waiting clipped."""
    x = float(max(int(w_us), 0)) / 1e6
    y = alpha * x
    y = y + beta
    return beta if beta <= y else y


def tuf0_seconds(beta: float, alpha: float, ert_s: float, t_s: float) -> float:
    """Plain real-valued Eq. 1 (used only by pins that quote seconds)."""
    return min(beta, alpha * (t_s - ert_s) + beta)
