"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9}.get(u, 1.0)
        per[r[idi]][r[mi]] = v * scale
        names[r[idi]] = r[ki].split("(")[0].replace("void ", "")[:48]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'us':>10} {'share':>6} {'n':>5} {'GB/s':>7}  kernel")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {100 * t / tot:5.1f}% {n:5d} {b / max(t, 1e-9) / 1e3:7.0f}  {k}")
    print(f"{tot:10.1f} total us")


if __name__ == "__main__":
    main(sys.argv[1])
