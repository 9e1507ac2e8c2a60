"""Per-kernel roofline table from an ncu --csv metrics log (time, DRAM bytes,
tensor / fp64 pipe activity, SM-time):

    python tools/kernel_roofline.py log.csv [--traffic-json profiles/roofline_traffic.json CFG]

--traffic-json merges {CFG: {kernel: DRAM bytes per launch}} into the given
file; bench.py reads roofline.traffic from it (per config, per kernel)."""
import collections
import csv
import json
import os
import sys

_PEAKS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
try:
    HBM = float(json.load(open(_PEAKS))["hbm_gbs"])   # GB/s, measured copy kernel
except Exception:
    HBM = 6650.0                                      # B200_PROFILING.md fallback

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), \
    h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "%": 1, "cycle": 1, "": 1}
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        per[(r[0], r[ki])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    except ValueError:  # "n/a" (metric not collected for this launch)
        continue
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for (_, k), m in per.items():
    name = k.split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")[:58]
    a = agg[name]
    a["n"] += 1
    t = m.get("gpu__time_duration.sum", 0.0)
    a["t"] += t
    a["bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a["tensor"] += t * m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
    a["fp64"] += t * m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
    a["smc"] += m.get("sm__cycles_active.sum", 0.0)
tot = sum(a["t"] for a in agg.values())
print(f"total {tot * 1e3:.2f} ms over {len(per)} launches\n")
print("| kernel | launches | ms | share | DRAM MB | GB/s | % HBM | tensor pipe % | fp64 pipe % |")
print("|---|---|---|---|---|---|---|---|---|")
for name, a in sorted(agg.items(), key=lambda x: -x[1]["t"])[:24]:
    gbs = a["bytes"] / a["t"] / 1e9 if a["t"] else 0.0
    print(f"| `{name}` | {int(a['n'])} | {a['t'] * 1e3:.3f} | {a['t'] / tot * 100:.1f}% | "
          f"{a['bytes'] / 1e6:.1f} | {gbs:.0f} | {gbs / HBM * 100:.1f} | "
          f"{a['tensor'] / a['t']:.1f} | {a['fp64'] / a['t']:.1f} |")

if "--traffic-json" in sys.argv:
    i = sys.argv.index("--traffic-json")
    path, cfg = sys.argv[i + 1], sys.argv[i + 2]
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[cfg] = {name: a["bytes"] / a["n"] for name, a in agg.items()}
    # template kernels: also one entry per base name over all instantiations
    base = collections.defaultdict(lambda: [0.0, 0.0])
    for name, a in agg.items():
        b = name.replace("void ", "").split("<")[0]
        base[b][0] += a["bytes"]
        base[b][1] += a["n"]
    for b, (by, cnt) in base.items():
        if b and b not in data[cfg]:
            data[cfg][b] = by / cnt
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
