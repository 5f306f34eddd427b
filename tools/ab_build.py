"""A/B builds of the library with extra nvcc defines into ab/<name>/librt_b200.so (git-ignored;
travels to the GPU box with the snapshot).  Select one at run time with RT_LIB_PATH.
Usage: ab_build.py name [-DFOO=1 ...] [gemm_tc.cu=/path/to/other/gemm_tc.cu ...]"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_18695_b200 import build as B  # noqa: E402


def main():
    name = sys.argv[1]
    defs = [a for a in sys.argv[2:] if "=" not in a or a.startswith("-")]
    subst = dict(a.split("=", 1) for a in sys.argv[2:] if "=" in a and not a.startswith("-"))
    out = os.path.join(ROOT, "ab", name)
    os.makedirs(out, exist_ok=True)

    def comp(src):
        o = os.path.join(out, src.replace(".cu", ".o"))
        r = subprocess.run([B.NVCC] + B.FLAGS + defs + ["-c", subst.get(src, os.path.join(B.CSRC, src)), "-o", o],
                           capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stdout + r.stderr)
        return o

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, B.SOURCES))
    lib = os.path.join(out, "librt_b200.so")
    subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-o", lib]
                   + objs + ["-ldl", "-lpthread"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
