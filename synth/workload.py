"""Programmable workload composition (§6; tab:data_sample
PAPER.md:449-463; SURVEY AMB-21).

Events arrive as a Poisson process with rate EPS (events/s); each event spawns
U[1, Max TPE] tasks, each on a distinct agent (round-robin cursor), trace drawn
uniformly from the pool.  Times are integer microseconds (AMB-23).
Deterministic in ``seed``.
"""
from dataclasses import dataclass
import numpy as np

from .traces import make_trace
from .vocab import SkillVocab


@dataclass
class Request:
    ordinal: int
    agent_id: int
    arrival_us: int
    trace_id: int
    prompt: np.ndarray
    plan: np.ndarray
    beta: float
    alpha: float
    ert_us: int
    exec_window_us: int

    @property
    def max_new_tokens(self) -> int:
        return int(len(self.plan))


def _mk(ordinal, agent, arrival, tid, vocab, seed, prompt_len_range, plan_len, exec_window_us):
    rng = np.random.Generator(np.random.PCG64([seed, 7919, ordinal]))
    pl = None
    if prompt_len_range is not None:
        lo, hi = prompt_len_range
        pl = int(rng.integers(lo, hi + 1))
    tr = make_trace(tid, vocab, seed=seed * 1000003 + ordinal, prompt_len=pl, plan_len=plan_len)
    return Request(ordinal, agent, int(arrival), tid, tr.prompt, tr.plan, tr.beta, tr.alpha,
                   tr.ert_us, exec_window_us)


def compose_workload(n_agents: int, eps: float, max_tpe: int, trace_pool, duration_s: float,
                     seed: int, vocab: SkillVocab, prompt_len_range=None, plan_len=None,
                     exec_window_us: int = 90000, max_requests=None):
    """Open-loop Poisson composition; returns requests sorted by (arrival, ordinal)."""
    rng = np.random.Generator(np.random.PCG64([seed, 1]))
    t = 0.0
    out = []
    cursor = 0
    pool = list(trace_pool)
    while True:
        t += rng.exponential(1.0 / eps)
        if t >= duration_s:
            break
        n = int(rng.integers(1, max_tpe + 1))
        n = min(n, n_agents)  # excess tasks dropped
        t_us = int(t * 1e6)
        for _ in range(n):
            tid = pool[int(rng.integers(0, len(pool)))]
            agent = cursor % n_agents
            cursor += 1
            out.append(_mk(len(out), agent, t_us, tid, vocab, seed, prompt_len_range, plan_len,
                           exec_window_us))
            if max_requests is not None and len(out) >= max_requests:
                return out
    return out


def closed_loop_requests(agent_id: int, ordinal: int, arrival_us: int, trace_pool, seed: int,
                         vocab: SkillVocab, prompt_len_range=None, plan_len=None,
                         exec_window_us: int = 90000) -> Request:
    """Saturation mode: the agent's next request after its previous one completed."""
    rng = np.random.Generator(np.random.PCG64([seed, 2, agent_id, ordinal]))
    pool = list(trace_pool)
    tid = pool[int(rng.integers(0, len(pool)))]
    return _mk(ordinal, agent_id, arrival_us, tid, vocab, seed, prompt_len_range, plan_len,
               exec_window_us)
