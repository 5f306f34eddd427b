"""In-pipeline kernel timeline of the bench step from the device trace (RT_FLAG_TRACE).

Per launch (grouped by %gridid): `lead` = first CTA entry -> first CTA past its
dependency wait (how early PDL let it start), `gap` = previous launch's last CTA exit ->
this launch's first ready CTA (dependency / launch latency on the critical path),
`body` = first ready -> last exit.  Aggregated per kernel role over the traced steps."""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import bench  # noqa: E402
import profile_step  # noqa: E402
from paper_2412_18695_b200 import rt  # noqa: E402

CLOCK_GHZ = 1.965   # SM clock under load (bench clocks line) for the clock64 phase marks
EPI = {0: "store", 1: "lm_head", 2: "qkv", 3: "resid", 4: "swiglu", 5: "part"}


def role(kind, layer_pos):
    base = kind & 0xFF
    if base == 1:
        mode = (kind >> 8) & 0xFF
        name = EPI.get(mode, str(mode))
        if mode == 3:   # O projection or down projection: alternate within a layer
            name = "o_proj" if layer_pos == 0 else "down"
        if mode == 5:   # raw split-K partials: QKV, O, down in layer order
            name = ("qkv", "o_proj", "down")[layer_pos] + "(part)"
        return f"gemm_{name}(S={kind >> 16})"
    return rt.TRACE_KINDS.get(base, str(base))


def analyse(tr):
    launches = collections.OrderedDict()
    phases = collections.defaultdict(list)
    for r in np.sort(tr, order="t_entry"):
        g = int(r["grid"])
        if int(r["kind"]) & 0x80:      # GEMM phase marks of one CTA
            phases[g].append((int(r["t_entry"]), int(r["t_ready"]), int(r["t_aux"]), int(r["t_exit"])))
            continue
        if g not in launches:
            launches[g] = dict(grid=g, kind=int(r["kind"]), entry=int(r["t_entry"]), ready=int(r["t_ready"]),
                               exit=int(r["t_exit"]), ctas=0, main=[], epi=[])
        L = launches[g]
        L["ready"] = min(L["ready"], int(r["t_ready"]))
        L["exit"] = max(L["exit"], int(r["t_exit"]))
        L["ctas"] += 1
        if r["t_aux"]:
            L["main"].append((int(r["t_aux"]) - int(r["t_ready"])) / 1e3)
            L["epi"].append((int(r["t_exit"]) - int(r["t_aux"])) / 1e3)
    seq = sorted(launches.values(), key=lambda L: L["entry"])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0, [], []])
    ph_agg = collections.defaultdict(list)
    resid_seen = 0
    prev_role = None
    prev_exit = None
    for L in seq:
        pos = 0
        if (L["kind"] & 0xFF) == 1 and ((L["kind"] >> 8) & 0xFF) == 3:
            pos = resid_seen % 2
            resid_seen += 1
        if (L["kind"] & 0xFF) == 1 and ((L["kind"] >> 8) & 0xFF) == 5:
            # raw partials: O follows the attention, down follows gate/up, QKV otherwise
            pos = 1 if prev_role == "attn" else (2 if (prev_role or "").startswith("gemm_swiglu") else 0)
        name = role(L["kind"], pos)
        prev_role = name
        gap = (L["ready"] - prev_exit) / 1e3 if prev_exit is not None else 0.0
        a = agg[name]
        a[0] += 1
        a[1] += (L["ready"] - L["entry"]) / 1e3
        a[2] += gap
        a[3] += (L["exit"] - L["ready"]) / 1e3
        a[4] += L["ctas"]
        if L["main"]:
            a[5].append(float(np.median(L["main"])))
            a[6].append(float(np.median(L["epi"])))
        if L["grid"] in phases:
            p = np.array(phases[L["grid"]], dtype=np.float64)
            p = p.astype(np.uint64)
            cyc = np.stack([f for k in range(4) for f in (p[:, k] & 0xFFFFFFFF, p[:, k] >> 32)], axis=1)
            ph_agg[name].append(np.median(cyc.astype(np.float64), axis=0) / CLOCK_GHZ / 1e3)
        prev_exit = max(prev_exit or 0, L["exit"])
    span = (max(L["exit"] for L in seq) - min(L["entry"] for L in seq)) / 1e3
    return agg, span, len(seq), ph_agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--agents", type=int, default=None)
    ap.add_argument("--workload", default="C3", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--gemm-path", type=int, default=0)
    ap.add_argument("--json", default=None)
    ap.add_argument("--raw", default=None, help="save the raw per-CTA records (.npy)")
    a = ap.parse_args()
    eng, now = profile_step.setup(a.agents, flags=rt.RT_FLAG_TRACE, workload=a.workload, gemm_path=a.gemm_path)
    eng.reset_stats()
    for _ in range(a.steps):
        info = eng.step(now())
    eng.sync()
    print("last round:", {k: info[k] for k in ("n_running", "n_waiting", "n_admitted", "n_refused_mem", "n_refused_wcet")})
    tr = eng.trace()
    if a.raw:
        np.save(a.raw, tr)
    agg, span, n, ph = analyse(tr)
    print(f"{n} launches, {len(tr)} CTA records, span {span:.1f} us over {a.steps} steps "
          f"({span / a.steps:.1f} us/step incl. host gaps between steps)")
    print(f"{'role':28s} {'n':>5s} {'lead us':>8s} {'gap us':>8s} {'body us':>8s} {'sum us/step':>12s}"
          f" {'cta main':>9s} {'cta epi':>8s}")
    rows = []
    for name, (cnt, lead, gap, body, ctas, mains, epis) in sorted(agg.items(),
                                                                 key=lambda x: -(x[1][2] + x[1][3])):
        per_step = (gap + body) / a.steps
        mm = float(np.median(mains)) if mains else float("nan")
        me = float(np.median(epis)) if epis else float("nan")
        print(f"{name:28s} {cnt:5d} {lead / cnt:8.2f} {gap / cnt:8.2f} {body / cnt:8.2f} {per_step:12.1f}"
              f" {mm:9.2f} {me:8.2f}")
        rows.append(dict(role=name, launches=cnt, lead_us=lead / cnt, gap_us=gap / cnt, body_us=body / cnt,
                         us_per_step=per_step, ctas=ctas // cnt, cta_main_us=mm, cta_epilogue_us=me))
    print("GEMM epilogue phases after the accumulator is complete (median us at 1.965 GHz): park | "
          "cluster barrier | slices received | partials loaded | - | epilogue loop | final reduction | bulk-copy drain")
    for name, v in ph.items():
        if name.startswith("sched"):
            continue
        m = np.median(np.array(v), axis=0)
        print(f"  {name:28s} " + " ".join(f"{x:7.2f}" for x in m))
    for name, v in ph.items():
        if name.startswith("sched"):
            m = np.median(np.array(v), axis=0)
            print(f"{name} phases (median us): ingest | score | sort | wcet+candidates | admit | assemble | "
                  "page pops | rows + publish")
            print("  " + " ".join(f"{x:7.2f}" for x in m))
    if a.json:
        json.dump(dict(steps=a.steps, span_us=span, launches=n, roles=rows), open(a.json, "w"), indent=1)
    eng.close()


if __name__ == "__main__":
    main()
