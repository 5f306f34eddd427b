"""Scripted robot plans shaped like the paper's trace library (tab:task_list,
PAPER.md:417-445; SURVEY §8d "Traces (scripted)").

| class        | trace ids | prompt | plan                              | TUF  |
| drone-normal | 1-5       | 1300   | 20 tokens, 3-4 skills             | beta 1, alpha -2, ERT 1 s    |
| drone-urgent | 6-8       | 1300   | 13 tokens, 1-2 skills             | beta 2, alpha -6.67, ERT 0.2 s |
| arm          | 9-11      | 2884   | 100 tokens, skill every <=10 toks | normal               |

Prompt sizes: 170.35 MB / 128 KiB per token = 1300; 2884 from
tab:latency.  Plan lengths: "around 100 tokens compared to the
20-token outputs".  Trace 2 (task type 1) plans print-like 1 ms
skills.  The plan always ends with EOS.  Non-skill "filler"
tokens are seeded random ids below the skill block.
"""
from dataclasses import dataclass
import numpy as np

from .vocab import SkillVocab

TUF_NORMAL = (1.0, -2.0, 1000000)     # (beta, alpha, ERT_us)
TUF_URGENT = (2.0, -6.67, 200000)     # PAPER.md:604 (alpha stored as printed, AMB-20)

TRACE_CLASSES = {
    1: "drone-normal", 2: "drone-normal", 3: "drone-normal", 4: "drone-normal", 5: "drone-normal",
    6: "drone-urgent", 7: "drone-urgent", 8: "drone-urgent",
    9: "arm", 10: "arm", 11: "arm",
}

_CLASS = {
    "drone-normal": dict(prompt=1300, plan=20, skills=(3, 4), tuf=TUF_NORMAL),
    "drone-urgent": dict(prompt=1300, plan=13, skills=(1, 2), tuf=TUF_URGENT),
    "arm": dict(prompt=2884, plan=100, skills=None, tuf=TUF_NORMAL),
}


@dataclass
class Trace:
    trace_id: int
    cls: str
    prompt: np.ndarray     # int32 prompt token ids
    plan: np.ndarray       # int32 scripted output tokens (ends with EOS)
    beta: float
    alpha: float
    ert_us: int

    @property
    def urgent(self) -> bool:
        return self.cls == "drone-urgent"


def _filler(vocab: SkillVocab, rng, n):
    return rng.integers(0, vocab.skill_begin, size=n, dtype=np.int64).astype(np.int32)


def make_plan(cls: str, trace_id: int, vocab: SkillVocab, rng, plan_len=None) -> np.ndarray:
    spec = _CLASS[cls]
    n = spec["plan"] if plan_len is None else int(plan_len)
    assert n >= 2
    plan = _filler(vocab, rng, n)
    plan[-1] = vocab.eos_id
    body = n - 1
    if cls == "arm":
        pool = vocab.skill_ids(["pick", "place"])
        # one skill in every window of 10 tokens (positions 10*i + r, r in [2, 9])
        pos = []
        for w in range(0, body, 10):
            hi = min(w + 10, body)
            lo = min(w + 2, hi - 1)
            pos.append(int(rng.integers(lo, hi)))
    else:
        if trace_id == 2:
            pool = vocab.skill_ids(["p", "iv"])
        else:
            pool = vocab.skill_ids(["mf", "mb", "ml", "mr", "mu", "md", "tc", "tu", "s"])
        lo, hi = spec["skills"]
        k = int(rng.integers(lo, hi + 1))
        k = max(1, min(k, body))
        pos = sorted(int(x) for x in rng.choice(np.arange(1, body + 1) - 1, size=k, replace=False))
    for p in pos:
        plan[p] = pool[int(rng.integers(0, len(pool)))]
    return plan


def system_prefix(vocab: SkillVocab, robot: str = "drone", n_tokens: int = 1216, seed: int = 0) -> np.ndarray:
    """The fixed part of a robot's prompt — skill set, guidance and examples, which PAPER.md:211
    says are pre-stored on the server — as seeded filler tokens; shared by every request of that
    robot type (DESIGN reading R-PFX: 1216 of the drone's 1300 prompt tokens = 76 pages, the
    last 84 are the task)."""
    rng = np.random.Generator(np.random.PCG64([seed, 0x5E5, len(robot)]))
    return _filler(vocab, rng, n_tokens)


def make_trace(trace_id: int, vocab: SkillVocab, seed: int, prompt_len=None, plan_len=None,
               prefix=None) -> Trace:
    """One scripted request of the given trace id; deterministic in ``seed``.  ``prefix``
    (optional): the prompt starts with these tokens and the rest is per-request filler."""
    cls = TRACE_CLASSES[trace_id]
    rng = np.random.Generator(np.random.PCG64([seed, trace_id]))
    spec = _CLASS[cls]
    pl = spec["prompt"] if prompt_len is None else int(prompt_len)
    if prefix is None:
        prompt = _filler(vocab, rng, pl)
    else:
        prefix = np.asarray(prefix, dtype=np.int32)
        prompt = np.concatenate([prefix, _filler(vocab, rng, pl - len(prefix))]).astype(np.int32)
    plan = make_plan(cls, trace_id, vocab, rng, plan_len)
    beta, alpha, ert = spec["tuf"]
    return Trace(trace_id, cls, prompt, plan, beta, alpha, ert)
