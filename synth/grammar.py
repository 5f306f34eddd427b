"""Synthetic multi-token vocabularies for the stop grammars (PAPER.md:206-207,
388: the stop checker detokenizes as it generates and matches executable skills with a regular
expression; chatbot sentence / paragraph segments).

Data only (no method arithmetic): every token id gets a TEXT (what a detokenizer would emit)
and a CLASS (rt.h RT_TC_*) for the device DFA; both describe the same tokens.

  skill names  class 1 + index, text " <name>"   (TypeFly-style names; the
                                                  leading space keeps a name a whole word)
  "(" ")" ";"  classes 80, 81, 82
  digits 0-9   classes 64 .. 73, text "0" .. "9"
  "." "!" "?"  class 91 (sentence end)
  "\\n\\n"     class 92 (paragraph end)
  EOS          V - 1, text ""
  other        class 90 (a word), text "w<id> "

Skill execution estimates (synthetic, as synth/vocab.py): E_min(name, arg) = base + unit * arg
with move 800000 + 20000 / cm, turn 500000 + 5000 / degree, p / iv 1000, s 2000000,
pick / place 3000000 (arg = object id).  Chatbot reading time: 300 words per minute
 = 200000 us per word.
"""
from dataclasses import dataclass
import numpy as np

from .vocab import SKILL_KINDS

TC_OTHER, TC_DIGIT0, TC_LPAREN, TC_RPAREN, TC_SEMI, TC_WORD, TC_SENT_END, TC_PARA_END = 0, 64, 80, 81, 82, 90, 91, 92
GRAMMAR_TOKEN, GRAMMAR_SKILL, GRAMMAR_SENTENCE, GRAMMAR_PARAGRAPH = 0, 1, 2, 3
MAX_SKILL_NAMES = 63
WORD_US = 200000  # 60 s / 300 words

_E = {"mf": (800000, 20000), "mb": (800000, 20000), "ml": (800000, 20000), "mr": (800000, 20000),
      "mu": (800000, 20000), "md": (800000, 20000), "tc": (500000, 5000), "tu": (500000, 5000),
      "iv": (1000, 0), "p": (1000, 0), "s": (2000000, 0), "pick": (3000000, 0), "place": (3000000, 0)}


@dataclass
class GrammarVocab:
    vocab: int
    eos_id: int
    tok_text: list              # str per token
    tok_class: np.ndarray       # int16 [V]
    skill_base_us: np.ndarray   # int32 [63]
    skill_unit_us: np.ndarray   # int32 [63]
    names: list                 # skill names (index = class - 1)
    ids: dict                   # text -> token id of every special token
    # single-token tables (unused by the grammars; keep the engine's TOKEN tables valid)
    tok_skill: np.ndarray = None
    tok_exec_min_us: np.ndarray = None
    words: tuple = (0, 0)       # [lo, hi) token ids of plain words


def make_grammar_vocab(vocab: int) -> GrammarVocab:
    assert vocab >= 128
    eos = vocab - 1
    text = [f"w{t} " for t in range(vocab)]
    cls = np.full(vocab, TC_WORD, dtype=np.int16)
    ids = {}
    t = eos - 1

    def put(s, c):
        nonlocal t
        text[t] = s
        cls[t] = c
        ids[s] = t
        t -= 1

    for i, n in enumerate(SKILL_KINDS):
        put(" " + n, 1 + i)
    put("(", TC_LPAREN)
    put(")", TC_RPAREN)
    put(";", TC_SEMI)
    for d in range(10):
        put(str(d), TC_DIGIT0 + d)
    for s in (".", "!", "?"):
        put(s, TC_SENT_END)
    put("\n\n", TC_PARA_END)
    text[eos] = ""
    cls[eos] = TC_OTHER
    base = np.zeros(MAX_SKILL_NAMES, dtype=np.int32)
    unit = np.zeros(MAX_SKILL_NAMES, dtype=np.int32)
    for i, n in enumerate(SKILL_KINDS):
        base[i], unit[i] = _E[n]
    return GrammarVocab(vocab, eos, text, cls, base, unit, list(SKILL_KINDS), ids,
                        tok_skill=np.full(vocab, -1, dtype=np.int16), tok_exec_min_us=np.zeros(vocab, dtype=np.int32),
                        words=(0, t + 1))


def statement(gv: GrammarVocab, name: str, arg=None):
    """Token ids of  name ( arg ) ;  (arg None: empty parentheses)."""
    toks = [gv.ids[" " + name], gv.ids["("]]
    if arg is not None:
        toks += [gv.ids[c] for c in str(int(arg))]
    return toks + [gv.ids[")"], gv.ids[";"]]


def robot_plan(gv: GrammarVocab, rng, n_stmts=3, words=(0, 3)):
    """A plan of skill statements with a few filler words before each, then EOS."""
    out = []
    for _ in range(n_stmts):
        out += [int(rng.integers(*gv.words)) for _ in range(int(rng.integers(*words)))]
        name = gv.names[int(rng.integers(0, 8))]
        arg = None if name in ("iv", "p") else int(rng.integers(1, 20)) * 10
        out += statement(gv, name, arg)
    return np.array(out + [gv.eos_id], dtype=np.int32)


def chat_text(gv: GrammarVocab, rng, n_par=2, n_sent=(2, 4), n_words=(3, 9)):
    """Paragraphs of sentences of words, ended by . ! ? and paragraph breaks, then EOS."""
    out = []
    ends = [gv.ids[s] for s in (".", "!", "?")]
    for _ in range(n_par):
        for _ in range(int(rng.integers(*n_sent))):
            out += [int(rng.integers(*gv.words)) for _ in range(int(rng.integers(*n_words)))]
            out.append(ends[int(rng.integers(0, 3))])
        out.append(gv.ids["\n\n"])
    return np.array(out + [gv.eos_id], dtype=np.int32)
