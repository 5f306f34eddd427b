"""Pins for the multi-token stop grammars (PAPER.md:206-207 detokenize as
generated, PAPER.md:388 regular-expression matching of robot actions, PAPER.md:606-609
chatbot sentence / paragraph segments read at 300 words per minute).

* The paper's example plan "mu(100);mf(50)", generated as the tokens
  " mu" "(" "1" "0" "0" ")" ";" " mf" "(" "5" "0" ")" ";" (13 tokens), ends two segments at the
  two ";" tokens with E_min(mu, 100) and E_min(mf, 50) — and a statement split by the 10-token
  CAP still completes in the next segment (the text buffer survives the boundary).
* Near misses never stop: missing ";" / ")", a word between the name and "(", a word that
  merely ends in a skill name, nested parentheses.
* Chatbot: sentence mode stops after every . ! ? (and paragraph end), paragraph mode only at
  paragraph ends, and a segment's execution estimate is 200 ms per word (60 s / 300 words).
* The grammars reduce to the same segment structure for the same text, so the method's
  mechanics (suspend / resume, token fidelity) are unchanged.
"""
import numpy as np
import pytest

from oracle.engine import (OracleEngine, STOP_SKILL, STOP_CAP, STOP_EOS, GRAMMAR_SKILL, GRAMMAR_SENTENCE,
                           GRAMMAR_PARAGRAPH)
from synth import engine_params
from synth.grammar import make_grammar_vocab, statement, robot_plan, chat_text, WORD_US


@pytest.fixture(scope="module")
def gv():
    return make_grammar_vocab(512)


def run(gv, plan, grammar, window=0, **kw):
    p = engine_params("paper-4090", max_ctx=256, n_pages=32, stop_grammar=grammar, **kw)
    e = OracleEngine(p, gv.tok_skill, gv.tok_exec_min_us, gv.eos_id, gv.vocab, grammar=gv)
    e.submit(0, [1, 2, 3], 0, 1_000_000, -2.0, 1.0, window, 0, script=list(plan))
    e.run_until_idle()
    return e.poll()


def test_paper_plan_mu100_mf50(gv):
    plan = statement(gv, "mu", 100) + statement(gv, "mf", 50) + [gv.eos_id]
    assert "".join(gv.tok_text[t] for t in plan) == " mu(100); mf(50);"
    segs = run(gv, plan, GRAMMAR_SKILL)
    assert [(s["tok_end"], s["reason"], s["n_skills"], s["est_exec_us"]) for s in segs] == [
        (7, STOP_SKILL, 1, 800000 + 20000 * 100), (13, STOP_SKILL, 1, 800000 + 20000 * 50), (14, STOP_EOS, 0, 0)]
    # window 10 s: both statements in one segment, ended by EOS
    segs = run(gv, plan, GRAMMAR_SKILL, window=10_000_000, max_seg_tokens=16)
    assert [(s["tok_end"], s["reason"], s["n_skills"]) for s in segs] == [(14, STOP_EOS, 2)]


def test_statement_split_by_cap_completes_later(gv):
    w = gv.words[0]
    plan = [w] * 7 + statement(gv, "tc", 90) + [gv.eos_id]      # 7 words + 6 tokens: crosses the 10-cap
    segs = run(gv, plan, GRAMMAR_SKILL)
    assert [(s["tok_end"], s["reason"]) for s in segs] == [(10, STOP_CAP), (13, STOP_SKILL), (14, STOP_EOS)]
    assert segs[1]["est_exec_us"] == 500000 + 5000 * 90 and segs[1]["n_skills"] == 1


@pytest.mark.parametrize("bad", [
    lambda gv: statement(gv, "mf", 50)[:-1],                                   # no ";"
    lambda gv: [t for t in statement(gv, "mf", 50) if t != gv.ids[")"]],       # no ")"
    lambda gv: [gv.ids[" mf"], gv.words[0]] + statement(gv, "mf", 5)[1:],       # word before "("
    lambda gv: [gv.ids[" mf"], gv.ids["("], gv.ids["("], gv.ids["5"], gv.ids[")"], gv.ids[";"]],
    lambda gv: [gv.ids["("], gv.ids["5"], gv.ids[")"], gv.ids[";"]],           # no name
])
def test_near_misses_do_not_stop(gv, bad):
    plan = bad(gv) + [gv.eos_id]
    segs = run(gv, plan, GRAMMAR_SKILL, max_seg_tokens=16)
    assert [s["reason"] for s in segs] == [STOP_EOS] and segs[0]["n_skills"] == 0


def test_empty_args_and_restart_on_name(gv):
    # " mf(5" interrupted by a new name: the later statement is the one completed
    plan = [gv.ids[" mf"], gv.ids["("], gv.ids["5"]] + statement(gv, "iv") + [gv.eos_id]
    segs = run(gv, plan, GRAMMAR_SKILL, max_seg_tokens=16)
    assert segs[0]["reason"] == STOP_SKILL and segs[0]["est_exec_us"] == 1000


def test_chat_sentence_and_paragraph(gv):
    rng = np.random.default_rng(0)
    text = chat_text(gv, rng, n_par=2, n_sent=(2, 3), n_words=(2, 4))
    ends = [i for i, t in enumerate(text) if gv.tok_text[t] in (".", "!", "?")]
    paras = [i for i, t in enumerate(text) if gv.tok_text[t] == "\n\n"]
    s_sent = run(gv, text, GRAMMAR_SENTENCE, max_seg_tokens=16)
    s_para = run(gv, text, GRAMMAR_PARAGRAPH, max_seg_tokens=16)
    cut = lambda segs: [s["tok_end"] - 1 for s in segs if s["reason"] == STOP_SKILL]  # noqa: E731
    assert cut(s_sent) == sorted(ends + paras)
    assert cut(s_para) == paras
    for segs in (s_sent, s_para):
        for s in segs:   # reading time = 200 ms per word of the segment
            assert s["est_exec_us"] == WORD_US * sum(1 for t in s["tokens"] if gv.tok_text[t].startswith("w"))
        assert sum((s["tokens"] for s in segs), []) == list(text)


def test_robot_plans_every_statement_is_a_boundary(gv):
    rng = np.random.default_rng(3)
    for _ in range(20):
        plan = robot_plan(gv, rng, n_stmts=3)
        segs = run(gv, plan, GRAMMAR_SKILL, max_seg_tokens=16)
        semis = [i for i, t in enumerate(plan) if t == gv.ids[";"]]
        assert [s["tok_end"] - 1 for s in segs if s["reason"] == STOP_SKILL] == semis
