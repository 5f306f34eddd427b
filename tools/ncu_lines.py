"""Warp-stall samples per CUDA source line (ncu --print-source cuda,sass), top lines."""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = {}
    fname = None
    h = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = r
            iall = h.index("Warp Stall Sampling (All Samples)")
            reasons = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
            continue
        if h is None or len(r) < len(h) or not r[0].isdigit():
            continue
        try:
            s = int(r[iall])
        except ValueError:
            continue
        if s == 0:
            continue
        key = (fname, int(r[0]))
        a = agg.setdefault(key, [0, r[1].strip()[:70], {}])
        a[0] += s
        for i, n in reasons:
            if r[i] not in ("0", ""):
                a[2][n] = a[2].get(n, 0) + int(r[i])
    tot = sum(a[0] for a in agg.values())
    print(tot, "samples")
    for (f, ln), (s, src, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        st = dict(sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f"{s:6d} {f}:{ln:<5d} {src:70s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
