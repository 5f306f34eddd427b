"""Eq. 4 PUD priority (oracle, test infrastructure only).

PAPER.md:308-320 (§4.3, Eq. 4):
    Pri(s_k, t) = [delta_k TUF_0(W(s_k; t)) + (1 - delta_k) TUF_1(W(s_k; t))] / (G(s_k) L(s_k))
    delta_k = 1 if k = 0 else 0.

Readings:
  AMB-2  W(s_k; t) = t + G + net - ref, ref = arrival (k=0) or end_est_{k-1} (k>0)
  AMB-3  L(s_k)    = max(eps_L, D - t - G), D = arrival + ERT (k=0) or end_est_{k-1}
  AMB-4  G         = constant g_us (PAPER.md:604, 90 ms)
  AMB-5  net       = net_us (PAPER.md:617, 8 ms)
  AMB-10 -0.0 canonicalised by `pri + 0.0`.
Exact op order (IEEE fp64, single rounding each, no FMA):
  num = TUF(...); a = g_us / 1e6; b = L_us / 1e6; den = a * b; pri = num / den; pri = pri + 0.0
"""
from .tuf import tuf0, tuf1


def waiting_estimate_us(t_us: int, g_us: int, net_us: int, ref_us: int) -> int:
    return int(t_us) + int(g_us) + int(net_us) - int(ref_us)


def slack_us(t_us: int, g_us: int, d_us: int, eps_l_us: int) -> int:
    return max(int(eps_l_us), int(d_us) - int(t_us) - int(g_us))


def priority(t_us, k, ref_us, d_us, ert_us, alpha, beta, g_us, net_us, eps_l_us) -> float:
    w = waiting_estimate_us(t_us, g_us, net_us, ref_us)
    if k == 0:
        num = tuf0(beta, alpha, ert_us, w)
    else:
        num = tuf1(beta, alpha, w)
    L = slack_us(t_us, g_us, d_us, eps_l_us)
    a = float(g_us) / 1e6
    b = float(L) / 1e6
    den = a * b
    pri = num / den
    return pri + 0.0


def priority_seconds(t, k, arrival, deadline, ert, alpha, beta, G, net, eps_l, prev_end=None):
    """Real-valued restatement used by pins quoting seconds."""
    ref = arrival if k == 0 else prev_end
    w = t + G + net - ref
    if k == 0:
        num = min(beta, alpha * (w - ert) + beta)
    else:
        num = min(beta, alpha * max(w, 0.0) + beta)
    L = max(eps_l, deadline - t - G)
    return num / (G * L)
