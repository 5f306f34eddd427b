"""Synthetic vocabularies with a token -> skill table (SURVEY §8d "Vocab / skills").

A random-init model has no tokenizer, so the paper's regex over
detokenized text (§5) is replaced by a table: each skill token id
is one ``(skill, parameter)`` pair, e.g. ``mf(50)`` (PAPER.md:28 plan
``mu(100);mf(50)``; TypeFly-style names PAPER.md:210).

E_min (the minimum execution-time estimate, §4.3) is a
SYNTHETIC input table: the paper gives no per-skill numbers except print ~1 ms
(PAPER.md:624).  Values (µs):
  move   = 800000 + 20000 * cm
  turn   = 500000 + 5000 * deg
  p / iv = 1000
  s      in {2,3,4} s, E_min 2 s  ("mode=Min -> 2.0 s")
  pick/place in {3,4,5} s, E_min 3 s
``realized`` lists the alternatives the agent simulator samples from
("randomly sample from this profiled data").
"""
from dataclasses import dataclass
import numpy as np

SKILL_KINDS = ["mf", "mb", "ml", "mr", "mu", "md", "tc", "tu", "iv", "p", "s", "pick", "place"]
K = {n: i for i, n in enumerate(SKILL_KINDS)}


@dataclass
class SkillVocab:
    vocab: int
    eos_id: int
    tok_skill: np.ndarray        # int16 [V]; -1 = not a skill
    tok_exec_min_us: np.ndarray  # int32 [V]; 0 for non-skills
    names: dict                  # tok -> "mf(50)"
    realized: dict               # tok -> tuple of realized durations (µs)
    skill_begin: int             # first skill id (contiguous block below EOS)

    def is_skill(self, tok: int) -> bool:
        return self.tok_skill[tok] >= 0

    def skill_ids(self, kinds=None):
        ids = [t for t in range(self.skill_begin, self.eos_id) if self.tok_skill[t] >= 0]
        if kinds is None:
            return ids
        ks = {K[k] for k in kinds}
        return [t for t in ids if int(self.tok_skill[t]) in ks]


def _entries(full: bool):
    ent = []
    cms = range(10, 201, 10) if full else range(20, 201, 20)
    degs = range(15, 361, 15) if full else range(45, 361, 45)
    for kind in ["mf", "mb", "ml", "mr", "mu", "md"]:
        for cm in cms:
            e = 800000 + 20000 * cm
            ent.append((kind, f"{kind}({cm})", e, (e,)))
    for kind in ["tc", "tu"]:
        for deg in degs:
            e = 500000 + 5000 * deg
            ent.append((kind, f"{kind}({deg})", e, (e,)))
    ent.append(("iv", "iv()", 1000, (1000,)))
    ent.append(("p", "p()", 1000, (1000,)))
    ent.append(("s", "s()", 2000000, (2000000, 3000000, 4000000)))
    objs = 16 if full else 4
    for kind in ["pick", "place"]:
        for o in range(objs):
            ent.append((kind, f"{kind}(obj{o})", 3000000, (3000000, 4000000, 5000000)))
    return ent


def make_vocab(vocab: int) -> SkillVocab:
    """Full table (203 ids) for V >= 4096, reduced table (87 ids) otherwise.

    EOS = V-1; skill ids occupy the contiguous block directly below EOS
    ([128052, 128255) for V=128256, [424, 511) for V=512).
    """
    full = vocab >= 4096
    ent = _entries(full)
    eos = vocab - 1
    begin = eos - len(ent)
    assert begin > 0
    tok_skill = np.full(vocab, -1, dtype=np.int16)
    tok_e = np.zeros(vocab, dtype=np.int32)
    names, realized = {}, {}
    for i, (kind, name, e, real) in enumerate(ent):
        t = begin + i
        tok_skill[t] = K[kind]
        tok_e[t] = e
        names[t] = name
        realized[t] = real
    return SkillVocab(vocab, eos, tok_skill, tok_e, names, realized, begin)
