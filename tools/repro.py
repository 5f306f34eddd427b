"""Small repro driver: 8B layer dims with few layers / requests (compute-sanitizer target)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import make_vocab, engine_params  # noqa: E402
from synth.configs import ModelShape  # noqa: E402
from synth.traces import make_trace  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--reqs", type=int, default=8)
ap.add_argument("--prompt", type=int, default=300)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--rows", type=int, default=4096)
ap.add_argument("--vocab", type=int, default=128256)
ap.add_argument("--gemm-path", type=int, default=0)
a = ap.parse_args()
shape = ModelShape("r", a.layers, 4096, 32, 8, 128, 14336, a.vocab)
v = make_vocab(shape.vocab)
B = max(64, a.reqs)
p = engine_params("b200-roofline", max_batch=B, max_tasks=2 * B, max_ctx=2048,
                  n_pages=max(2000, a.reqs * ((a.prompt + 40 + 15) // 16 + 1)))
eng = rt.Engine(shape, p, v, seed=1, max_rows_per_forward=a.rows, gemm_path=a.gemm_path)
for j in range(a.reqs):
    tr = make_trace(1 + j % 8, v, seed=j, prompt_len=a.prompt, plan_len=40)
    eng.submit(j, tr.prompt, 0, tr.ert_us, tr.alpha, tr.beta, 90000, script=tr.plan)
for i in range(a.steps):
    info = eng.step()
    eng.sync()
    print(i, info, flush=True)
print("ok")
