"""Aggregates an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def summarize(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
        name = r[ki].split("(")[0].replace("void ", "").replace("dmcg::", "").replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"total {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches",
           "| share | launches | total ms | avg us | kernel |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"| {v[1] / tot * 100:5.1f}% | {v[0]} | {v[1] / 1e3:.3f} | {v[1] / v[0]:.1f} | `{k[:70]}` |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20))
