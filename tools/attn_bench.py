"""Microbenchmark of the paged decode attention kernel at the C2-C5 operating points
(algorithmic bytes = attended tokens x K/V bytes + q + o, CUDA events, back-to-back)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402


def bench(B, ctx, nq=32, nkv=8, hd=128, iters=50, seed=0, ctxs=None):
    """ctxs (optional): per-row context lengths (max = ctx) in row order."""
    P = 16
    pages_per = (ctx + P - 1) // P
    n_pages = B * pages_per
    rng = np.random.default_rng(seed)
    perm = torch.from_numpy(rng.permutation(n_pages).astype(np.int32)).cuda()
    pt = perm.view(B, pages_per).contiguous()
    pool = torch.randn(n_pages * nkv * 64 * hd // 2, device="cuda").to(torch.bfloat16).view(torch.uint8)
    q = torch.randn(B, nq, hd, device="cuda").to(torch.bfloat16)
    row_task = torch.arange(B, dtype=torch.int32, device="cuda")
    if ctxs is None:
        ctxs = [ctx] * B
    row_sl = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    out = torch.empty(B, nq, hd, dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(rt.lib().rt_op_attention_ws_bytes(B, ctx, nq, hd) + 16, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        rt.paged_attention(q, pool, pt, row_task, row_sl, ctx, nq, nkv, hd, out, None, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        rt.paged_attention(q, pool, pt, row_task, row_sl, ctx, nq, nkv, hd, out, None, ws)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    alg = sum(ctxs) * nkv * hd * 2 * 2 + 2 * B * nq * hd * 2
    return us, alg / us / 1e3


def main():
    cases = [(64, 1310), (256, 2150), (128, 1310), (512, 280), (1, 4096), (4, 1310), (8, 1310), (16, 2884),
             (32, 2884), (64, 8192)]
    if len(sys.argv) > 1 and sys.argv[1] == "small":
        cases = [(1, 4096), (4, 1310), (8, 1310), (16, 2884), (32, 2884)]
    if len(sys.argv) > 1 and sys.argv[1] == "grid":   # B x ctx at 8B / 70B dims
        cases = [(b, c) for b in (8, 32, 64, 128, 256) for c in (512, 1310, 2884, 8192)]
    if len(sys.argv) > 1 and sys.argv[1] == "mixed":   # C3: 128 drone rows (1300) + 128 arm rows (2884)
        inter = [1300 if i % 2 == 0 else 2884 for i in range(256)]
        for name, cx in (("interleaved", inter), ("longest-first", sorted(inter, reverse=True)),
                         ("shortest-first", sorted(inter)), ("uniform", [2092] * 256)):
            us, gbs = bench(256, max(cx), ctxs=cx)
            print(f"C3 mix {name:15s}: {us:8.1f} us  {gbs:6.0f} GB/s", flush=True)
        return
    for B, ctx in cases:
        for nq in (32, 64):
            us, gbs = bench(B, ctx, nq=nq)
            print(f"B={B:4d} ctx={ctx:5d} G={nq // 8}: {us:8.1f} us  {gbs:6.0f} GB/s  "
                  f"({gbs / 6536:.3f} of 6536, {gbs / 8000:.3f} of 8000)", flush=True)


if __name__ == "__main__":
    main()
