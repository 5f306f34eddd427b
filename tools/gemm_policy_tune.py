"""Measure the prefill projection kernels per (shape, rows N) for every candidate (forced
tile width and CTA-pair kernel on / off through rt_op_gemm_tiled(path, bn)); one JSON line per
measurement.  `tools/gemm_policy_gen.py` turns the lines into the
dispatch table `paper_2412_18695_b200/csrc/gemm_policy.inc`."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)}
N_MAX = 4096


CANDIDATES = [(160, 0), (192, 0), (256, 0), (192, 1), (256, 1)]  # (tile width, CTA pair)


def main():
    import random
    rnd = random.Random(0)
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)
    for name in names:
        M, K = SHAPES[name]
        W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.bfloat16)
        Wt = torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda")
        rt.pack_tiled(W, Wt, M, K)
        del W
        cap = N_MAX + 256
        X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(N_MAX, M, device="cuda")
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        for N in range(160, N_MAX + 1, 32):
            # all candidates of one N back to back in random order (clocks drift with the
            # power state over a long sweep; a per-process sweep per width biased the choice)
            for bn, pair in rnd.sample(CANDIDATES, len(CANDIDATES)):
                path = rt.RT_GEMM_PATH_PAIR if pair else rt.RT_GEMM_PATH_STREAMK
                for _ in range(2):
                    rt.gemm_tiled(Wt, X, out, M, N, K, cap, 0, path=path, bn=bn)
                e0.record()
                for _ in range(8):
                    rt.gemm_tiled(Wt, X, out, M, N, K, cap, 0, path=path, bn=bn)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / 8 * 1e3
                print(json.dumps({"shape": name, "M": M, "K": K, "N": N, "bn": bn, "pair": pair, "us": round(us, 2)}),
                      flush=True)
        del Wt, X, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
