"""Run-to-run determinism of every projection path (rt_config.gemm_path): the same scripted rounds of a 512-row prefill at 8B dims, run 7 times per
path; prints the max |difference| of each run's logits against the first (all 0 when
deterministic)."""
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2412_18695_b200 import rt
from synth import MODEL_SHAPES, make_vocab, engine_params
from synth.configs import ModelShape
from synth.traces import make_trace
s8 = MODEL_SHAPES["llama3-8b"]
shape = ModelShape("sk", 2, s8.d_model, s8.n_q_heads, s8.n_kv_heads, s8.head_dim, s8.d_ff, s8.vocab)
v = make_vocab(shape.vocab)
p = engine_params("b200-roofline", max_batch=8, max_tasks=16, max_ctx=512, n_pages=8 * 32)
PATHS = {"auto": 0, "per_tile": 1, "hybrid": 2, "pair": 3, "decpair": 4}
def run(mode, prompt_len=64):
    eng = rt.Engine(shape, p, v, seed=23, flags=rt.RT_FLAG_KEEP_LOGITS, max_rows_per_forward=4096,
                    gemm_path=PATHS[mode])
    for a in range(8):
        tr = make_trace(1 + a, v, seed=a, prompt_len=prompt_len, plan_len=12)
        eng.submit(a, tr.prompt, 0, tr.ert_us, tr.alpha, tr.beta, 90000, script=tr.plan)
    logs = []
    for _ in range(4):
        info = eng.step(); B = info["n_running"]
        logs.append(eng.dump(rt.RT_DUMP_LOGITS, np.float32).reshape(B, -1).copy())
    eng.close()
    return logs
for mode in PATHS:
    ref = run(mode)
    for rep in range(6):
        got = run(mode)
        d = [float(np.abs(a - b).max()) for a, b in zip(ref, got)]
        print(mode, rep, ["%.3g" % x for x in d], flush=True)
