"""Epilogue phase profile of the tcgen05 projection kernel in isolation (device trace
bound through a scheduling-only engine with RT_FLAG_TRACE): isolated launches (sync
between) vs back-to-back launches, per shape and split."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402
from synth import make_vocab, engine_params  # noqa: E402

SHAPES = {"o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336), "qkv": (6144, 4096)}


def phases(tr):
    ph = tr[(tr["kind"] & 0x80) != 0]
    main = tr[((tr["kind"] & 0xFF) == 1)]
    cyc = np.stack([f for k in ("t_entry", "t_ready", "t_aux", "t_exit")
                    for f in (ph[k].astype(np.uint64) & 0xFFFFFFFF, ph[k].astype(np.uint64) >> 32)],
                   1).astype(np.float64) / 1965.0
    mainloop = (main["t_aux"].astype(np.int64) - main["t_ready"].astype(np.int64)) / 1e3
    epi = (main["t_exit"].astype(np.int64) - main["t_aux"].astype(np.int64)) / 1e3
    return np.median(cyc, 0), float(np.median(mainloop)), float(np.median(epi))


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    v = make_vocab(512)
    eng = rt.Engine(None, engine_params(max_batch=4, max_tasks=8, max_ctx=64, n_pages=16), v,
                    flags=rt.RT_FLAG_TRACE)
    for name, (M, K) in SHAPES.items():
        W = (torch.randn(M, K, device="cuda") * 0.02).to(torch.bfloat16)
        Wt = torch.empty(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda")
        rt.pack_tiled(W, Wt, M, K)
        cap = ((N + 255) // 256) * 256
        X = torch.randn(cap, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(N, M, device="cuda")
        for s in ([1, 2, 4, 8] if N <= 256 else [1]):
            if (K // 64) // s < 4:
                continue
            rt.gemm_tiled(Wt, X, out, M, N, K, cap, s)
            torch.cuda.synchronize()
            for mode in (["isolated", "back-to-back"] if N <= 256 else ["back-to-back"]):
                eng.reset_stats()
                for _ in range(10):
                    rt.gemm_tiled(Wt, X, out, M, N, K, cap, s)
                    if mode == "isolated":
                        torch.cuda.synchronize()
                torch.cuda.synchronize()
                trc = eng.trace()
                ph, ml, ep = phases(trc)
                main = trc[(trc["kind"] & 0xFF) == 1]
                span = (int(main["t_exit"].max()) - int(main["t_entry"].min())) / 1e3 / 10
                tf = 2.0 * M * N * K / (span * 1e-6) / 1e12
                print(f"{name:5s} N={N} S={s} {mode:13s} {span:8.1f} us/launch ({tf:6.0f} TF/s)  mainloop {ml:6.2f} us  "
                      f"epilogue {ep:6.2f} us  phases " + " ".join(f"{x:6.2f}" for x in ph), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
