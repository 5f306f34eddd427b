"""C5 per-GPU slice on one B200 (BASELINE.json configs[4]: 4096 agents, Llama-3-70B-shaped
layer dims, long multi-segment plans, KV retention stress on 8 x B200 -> 512 agents per GPU).

Llama-3-70B dims with all 80 layers (141 GB of bf16 weights), the KV pool in what is left of
HBM, 512 robot-arm agents with 128-token prompts and 256-token scripted plans (a skill every
<= 10 tokens: 20+ segments per request).  AMB-26 reservations (prompt + 256 new tokens = 24
pages of 5.2 MB) let only part of the agents hold KV at once: the rest are admission
refusals, and suspended requests keep their pages across segments (retention).  Reports
decode tok/s over K timed rounds (CUDA events on the engine stream), the running batch,
refusals, the pages held, and the tensor-bound ceiling of the step (2 x 69.5 G streamed
params x B tokens at the measured bf16 peak).  One JSON line.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params  # noqa: E402
from synth.traces import make_trace  # noqa: E402
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--agents", type=int, default=512)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--kv-gb", type=float, default=30.0)
    ap.add_argument("--layers", type=int, default=80)
    a = ap.parse_args()
    s7 = MODEL_SHAPES["llama3-70b"]
    from synth.configs import ModelShape
    shape = ModelShape("llama3-70b", a.layers, s7.d_model, s7.n_q_heads, s7.n_kv_heads, s7.head_dim, s7.d_ff,
                       s7.vocab)
    vocab = make_vocab(shape.vocab)
    page_bytes = shape.kv_bytes_per_token * 16
    n_pages = int(a.kv_gb * 1e9 // page_bytes)
    p = engine_params("b200-roofline", max_batch=a.agents, max_tasks=2 * a.agents, max_ctx=512, n_pages=n_pages,
                      clock_mode=1)
    t_create = time.perf_counter()
    eng = rt.Engine(shape, p, vocab, seed=77, flags=rt.RT_FLAG_TIMING, max_rows_per_forward=4096)
    t_create = time.perf_counter() - t_create
    t0 = time.perf_counter()

    def now():
        return int((time.perf_counter() - t0) * 1e6)

    for ag in range(a.agents):
        tr = make_trace(9 + ag % 3, vocab, seed=ag, prompt_len=128, plan_len=256)
        eng.submit(ag, tr.prompt, now(), tr.ert_us, tr.alpha, tr.beta, p.g_us, script=tr.plan)
    refused = 0
    t_fill = time.perf_counter()
    for _ in range(60):    # admissions up to the memory limit; prefill of the admitted prompts
        info = eng.step(now())
        refused += info["n_refused_mem"]
    eng.sync()
    t_fill = time.perf_counter() - t_fill
    eng.poll()
    eng.set_timing(False)
    eng.reset_stats()
    with bench.ClockSampler(0) as clk:
        lo = time.perf_counter()
        eng.mark(0)
        tok = 0
        bs = []
        for _ in range(a.steps):
            info = eng.step(now())
            tok += info["n_running"]
            bs.append(info["n_running"])
            refused += info["n_refused_mem"]
        eng.mark(1)
        ms = eng.elapsed_ms()
        clk.window(lo, time.perf_counter())
    segs = eng.poll()
    tasks = eng.tasks()
    held = int(tasks[(tasks[:, 1] == 1) | (tasks[:, 1] == 2)][:, 4].sum())
    waiting = int(((tasks[:, 1] == 1) & (tasks[:, 4] == 0)).sum())
    suspended_holding = int(((tasks[:, 1] == 1) & (tasks[:, 4] > 0)).sum())
    pk = bench.peaks()
    B = float(np.mean(bs))
    flops = 2.0 * (shape.weight_bytes_streamed() / 2) * B
    ceil_ms = flops / (pk.get("bf16_tflops_sustained", 1368.3) * 1e12) * 1e3
    out = {"config": f"C5 slice: {a.agents} robot-arm agents, llama3-70b dims x {a.layers} layers, 128-token prompts, "
                     "256-token scripted plans, AMB-26 reservations (24 pages per request)",
           "decode_tok_s": tok / (ms / 1e3), "ms_per_round": ms / a.steps, "mean_running": B,
           "tensor_bound_ms_per_round": ceil_ms, "frac_of_tensor_bound": ceil_ms / (ms / a.steps),
           "kv_pool_pages": n_pages, "kv_pool_gb": n_pages * page_bytes / 1e9, "pages_held": held,
           "refusals_mem": refused, "waiting_without_pages": waiting, "suspended_holding_pages": suspended_holding,
           "segments_in_timed_rounds": len(segs), "create_s": t_create, "fill_s": t_fill, "clocks": clk.summary()}
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()
