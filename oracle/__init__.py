"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct implementation of what the B200 hot path
computes, written from the paper (arxiv 2412.18695, /root/reference/PAPER.md)
in the paper's order and notation.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
(``paper_2412_18695_b200``) never imports it and shares no code with it; the
only shared module is ``synth/`` (seeded inputs, no method arithmetic).

Floating point is IEEE fp64 (Python floats / numpy float64, never FMA)
except where the method fixes bf16 materialisation points (c1 model).

Module map:
  tuf.py        c6   Eq. 1 TUF0 and TUF1
  priority.py   c7   Eq. 4 PUD priority
  bf16.py       —    bf16 RNE rounding (materialisation)    (pinned vs torch, P12)
  weights.py    c1   counter-based random init (AMB-15)     (pinned: statistics + closed form)
  model.py      c1   Llama decoder step, attention          (pinned vs HF transformers P7, SDPA P6)
  engine.py     c2,c3,c4,c8,c9  round loop: admission, paging, stop checker, retire
  agents.py     c5,c10  agent timeline + metrics
  bruteforce.py c12  Eq. 3 brute force + Theorem 1 check
  merge.py      c13  global top-K merge                     (set identity P13)

Parity pins: see tests/test_oracle_*.py; readings: DESIGN.md §Readings.
Unpinned: the exact intra-round order of c9 is a reading (DESIGN.md R-ROUND),
"parity unpinned" beyond the hand-worked traces in tests/golden/.
"""
