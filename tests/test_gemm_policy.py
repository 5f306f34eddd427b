"""The committed prefill-projection dispatch table is exactly what the generator makes of the
committed measurements (tools/gemm_policy_gen.py <- profiles/r01_gemm_policy_tune.jsonl), and
every bucket's choice is the fastest measured candidate."""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gemm_policy_gen as gen  # noqa: E402


def test_table_regenerates(tmp_path):
    out = tmp_path / "p.inc"
    gen.main(gen.SRC, str(out))
    assert out.read_text() == open(gen.DST).read()


def test_table_choices_are_fastest():
    meas = collections.defaultdict(dict)
    for line in open(gen.SRC):
        r = json.loads(line)
        meas[(r["M"], r["K"], r["N"])][(r["bn"], r["pair"])] = r["us"]
    rows = [l for l in open(gen.DST) if l.strip().startswith("{") and '"' in l]
    assert len(rows) == 4
    for l in rows:
        M, K, n_max = (int(v) for v in l.strip().strip("{},").split(",")[:3])
        code = l.split('"')[1]
        for j, ch in enumerate(code):
            N = 160 + 32 * j
            c = int(ch)
            choice = (gen.WIDTHS[c % 3], c // 3)
            d = meas[(M, K, N)]
            assert d[choice] == min(d.values())
        assert n_max == 160 + 32 * (len(code) - 1)
