"""Decode-projection microbenchmark per kernel path (rt_op_gemm_tiled with a forced path).

The four Llama-3-8B projections at N rows, each timed over launches that cycle through 8
distinct weight copies (3.5 GB in total at 8B dims, > the 126 MB L2: every launch streams its
weights from HBM, as in the decode step).  Prints us per launch and weight GB/s per path:
auto (the engine's dispatch), splitk (k_gemm_tc), streamk (k_gemm_sk), pair (k_gemm_2sm),
decpair (k_gemm_dec).  Usage: proj_bench.py [N ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)}
PATHS = {"auto": 0, "splitk": 1, "streamk": 2, "pair": 3, "decpair": 4}
COPIES = int(os.environ.get("PROJ_COPIES", "8"))  # 1: weights stay L2-resident between launches


def main():
    Ns = [int(a) for a in sys.argv[1:]] or [256]
    ws = {}
    for name, (M, K) in SHAPES.items():
        lst = []
        for c in range(COPIES):
            Wt = torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda")
            Wt.normal_(0, 0.02)
            lst.append(Wt)
        ws[name] = lst
    for N in Ns:
        cap = ((N + 255) // 256) * 256
        for name, (M, K) in SHAPES.items():
            X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
            out = torch.empty(N, M, device="cuda")
            cells = []
            for pname, path in PATHS.items():
                try:
                    for i in range(COPIES):
                        rt.gemm_tiled(ws[name][i], X, out, M, N, K, cap, 0, path=path)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    it = max(32, 4 * COPIES)
                    e0.record()
                    for i in range(it):
                        rt.gemm_tiled(ws[name][i % COPIES], X, out, M, N, K, cap, 0, path=path)
                    e1.record()
                    torch.cuda.synchronize()
                    us = e0.elapsed_time(e1) / it * 1e3
                    cells.append(f"{pname}:{us:6.1f}us/{M * K * 2 / us / 1e3:5.0f}GB/s")
                except Exception as ex:  # noqa: BLE001
                    cells.append(f"{pname}:ERR {ex}")
            # cuBLAS reference (torch.nn.functional.linear, bf16 out) on row-major copies
            try:
                Wr = [w[:M * K].view(M, K) for w in ws[name]]
                Xn = X[:N]
                for i in range(COPIES):
                    torch.nn.functional.linear(Xn, Wr[i])
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                it = max(32, 4 * COPIES)
                e0.record()
                for i in range(it):
                    torch.nn.functional.linear(Xn, Wr[i % COPIES])
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / it * 1e3
                cells.append(f"cublas:{us:6.1f}us/{M * K * 2 / us / 1e3:5.0f}GB/s")
            except Exception as ex:  # noqa: BLE001
                cells.append(f"cublas:ERR {ex}")
            print(f"N={N} {name:5s} " + "  ".join(cells), flush=True)


if __name__ == "__main__":
    main()
