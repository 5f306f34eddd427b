"""Decode-round throughput at SURVEY §8(d) C3 (one B200): 256 agents, half drone (traces 1-8,
1300-token prompts) and half robot arm (traces 9-11, 2884-token prompts), Llama-3-8B-shaped
random-init bf16, every context resident (private prompts, no prefix sharing, so algorithmic
attention bytes = HBM bytes), B_max 256.  Same two passes as bench.py: K rounds without
per-kernel events (tok/s, seg/s), then K rounds with CUDA events around every attention
launch (attention GB/s vs MEASURED_PEAKS).  One JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params  # noqa: E402
from synth.traces import make_trace  # noqa: E402
import bench  # noqa: E402


def main(K=10, W=3, B=256):
    shape = MODEL_SHAPES["llama3-8b"]
    vocab = make_vocab(shape.vocab)
    max_ctx = 4096
    plan_len = W + 2 * K + 16
    n_pages = (B // 2) * ((1300 + plan_len + 15) // 16 + 2) + (B // 2) * ((2884 + plan_len + 15) // 16 + 2)
    p = engine_params("b200-roofline", max_batch=B, max_tasks=2 * B, max_ctx=max_ctx, n_pages=n_pages, clock_mode=1)
    eng = rt.Engine(shape, p, vocab, seed=1234, flags=rt.RT_FLAG_TIMING, max_rows_per_forward=8192)
    t0 = time.perf_counter()

    def now():
        return int((time.perf_counter() - t0) * 1e6)

    for a in range(B):
        tid = 1 + (a * 7) % 8 if a % 2 == 0 else 9 + (a // 2) % 3
        tr = make_trace(tid, vocab, seed=a, plan_len=plan_len)
        eng.submit(a, tr.prompt, now(), tr.ert_us, tr.alpha, tr.beta, p.g_us, script=tr.plan)
    t_setup = time.perf_counter()
    for _ in range(400):
        info = eng.step(now())
        if info["n_running"] == B and info["n_prefill_rows"] == 0:
            break
    eng.sync()
    prefill_s = time.perf_counter() - t_setup
    assert info["n_running"] == B, info
    ctx = eng.tasks()
    for _ in range(p.speed_window + 1 + W):
        eng.step(now())
    eng.poll()
    eng.sync()
    eng.set_timing(False)
    eng.reset_stats()
    torch.cuda.synchronize()
    with bench.ClockSampler(0) as clk:
        time.sleep(0.05)
        lo = time.perf_counter()
        eng.mark(0)
        tok = 0
        for _ in range(K):
            tok += eng.step(now())["n_running"]
        eng.mark(1)
        ms = eng.elapsed_ms()
        clk.window(lo, time.perf_counter())
    segs = len(eng.poll())
    eng.set_timing(True)
    eng.reset_stats()
    for _ in range(K):
        eng.step(now())
    eng.sync()
    eng.step(now())
    eng.sync()
    st = eng.stats()
    pk = bench.peaks()
    gbs = st["attn_bytes"] / (st["attn_ms"] / 1e3) / 1e9
    out = {"config": "C3: 256 agents (128 drone ctx ~1300 + 128 arm ctx ~2884), llama3-8b-shape, B_max 256, "
                     "private prompts, contexts resident",
           "decode_tok_s": tok / (ms / 1e3), "segments_per_s": segs / (ms / 1e3), "ms_per_round": ms / K,
           "attention": {"achieved_gbs": gbs, "peak_gbs": pk["hbm_gbs"], "frac": gbs / pk["hbm_gbs"],
                         "frac_of_8000": gbs / 8000.0, "alg_bytes_per_launch": st["attn_bytes"] / st["attn_launches"],
                         "us_per_launch": st["attn_ms"] / st["attn_launches"] * 1e3},
           "kv_gb_per_round": st["attn_bytes"] / max(st["rounds"], 1) / 1e9,
           "prefill_s": prefill_s, "steps": K, "warmup": W, "clocks": clk.summary(),
           "mean_ctx": float(ctx[ctx[:, 0] >= 0][:, 3].mean()) if len(ctx) else None}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
