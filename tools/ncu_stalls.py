"""Top SASS lines by warp-stall samples of an ncu report's source page (with reasons)."""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
    h = rows[hi]
    ia, isrc = h.index("Address"), h.index("Source")
    iall = h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ri = [h.index(c) for c in reasons]
    data = []
    tot_r = {}
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[iall] in ("0", ""):
            continue
        st = {reasons[k][6:]: int(r[i]) for k, i in enumerate(ri) if r[i] not in ("0", "")}
        for k, v in st.items():
            tot_r[k] = tot_r.get(k, 0) + v
        data.append((int(r[iall]), r[ia][-5:], r[isrc].strip()[:64], st))
    tot = sum(d[0] for d in data)
    print(f"{tot} samples; by reason:", dict(sorted(tot_r.items(), key=lambda x: -x[1])))
    for d in sorted(data, key=lambda x: -x[0])[:top]:
        print(f"{d[0]:6d} {d[1]} {d[2]:64s} {d[3]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
