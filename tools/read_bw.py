"""HBM read ceiling of the decode attention's pattern (tools/bw/read_bw.cu): 8 KiB blocks by
cp.async.bulk into per-warp rings, no math, pages in pool order or shuffled.
Prints GB/s per (ring depth, CTAs per SM, order)."""
import ctypes
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "bw", "read_bw.cu")
SO = os.path.join(HERE, "bw", "read_bw.so")


def build():
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                        SRC, "-o", SO], check=True)
    return ctypes.CDLL(SO)


def main():
    lib = build()
    n_pages = 2 * 1024 * 1024 * 1024 // 8192 * 2  # 4 GB of 8 KiB blocks
    pool = torch.empty(n_pages * 8192, dtype=torch.uint8, device="cuda")
    pool.random_(0, 255)
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    orders = {"seq": torch.arange(n_pages, dtype=torch.int32, device="cuda"),
              "shuffled": torch.randperm(n_pages, device="cuda").to(torch.int32)}
    for oname, pages in orders.items():
        for stages in (3, 4, 6):
            for per_sm in (1, 2):
                if stages * 4 * 8192 * per_sm > 220 * 1024:
                    continue
                ctas = 148 * per_sm
                f = lambda: lib.read_bw(ctypes.c_void_p(pool.data_ptr()), ctypes.c_void_p(pages.data_ptr()), n_pages,
                                        ctas, stages, ctypes.c_void_p(sink.data_ptr()), None)
                for _ in range(3):
                    f()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for _ in range(10):
                    f()
                e1.record()
                torch.cuda.synchronize()
                s = e0.elapsed_time(e1) / 10 / 1e3
                print(f"{oname:8s} stages={stages} ctas/SM={per_sm}: {n_pages * 8192 / s / 1e9:7.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
