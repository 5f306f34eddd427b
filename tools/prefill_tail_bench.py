"""Prefill attention at the e2e operating point (bench `e2e`): R requests whose 1300-token
prompts share the drone's 1216-token registered prefix, so each prefills an 84-token tail
attending to ~1260 keys; 8B layer dims, 4 layers; device trace of the prefill round ->
k_attn_prefill time per layer (median over repeats)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params  # noqa: E402
from synth.configs import ModelShape  # noqa: E402
from synth.traces import make_trace, system_prefix  # noqa: E402


def main(R=4, reps=5):
    s8 = MODEL_SHAPES["llama3-8b"]
    shape = ModelShape("pf", 4, s8.d_model, s8.n_q_heads, s8.n_kv_heads, s8.head_dim, s8.d_ff, s8.vocab)
    v = make_vocab(shape.vocab)
    p = engine_params("b200-roofline", max_batch=64, max_tasks=256, max_ctx=2048, n_pages=64 * 130)
    eng = rt.Engine(shape, p, v, seed=3, flags=rt.RT_FLAG_TRACE, max_rows_per_forward=8192)
    pre = system_prefix(v, "drone", 1216, seed=0)
    eng.register_prefix(pre)
    times = []
    for rep in range(reps):
        for a in range(R):
            tr = make_trace(1, v, seed=rep * 100 + a, prompt_len=1300, plan_len=2, prefix=pre)
            eng.submit(a, tr.prompt, 0, tr.ert_us, tr.alpha, tr.beta, 90000, script=tr.plan)
        eng.sync()
        eng.reset_stats()
        info = eng.step()
        eng.sync()
        tr_ = eng.trace()
        for _ in range(4):
            eng.step()
        eng.poll()
        pf = tr_[(tr_["kind"] & 0xFF) == 10]
        by = {}
        for r in pf:
            g = int(r["grid"])
            lo, hi = by.get(g, (1 << 62, 0))
            by[g] = (min(lo, int(r["t_ready"])), max(hi, int(r["t_exit"])))
        per = [(hi - lo) / 1e3 for lo, hi in by.values()]
        times.append(float(np.median(per)))
        assert info["n_prefill_rows"] == R * 84, info
    print(f"R={R}: prefill attention {np.median(times):.1f} us per layer (84-token tails on a 1216 prefix)")


if __name__ == "__main__":
    for R in ([int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else (1, 4, 8)):
        main(R)
