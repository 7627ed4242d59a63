"""Summarises an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel launches, total and mean device time, share of the total."""
import collections
import csv
import sys


def summarise(path, steps=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        name = name.replace("void ", "").split("<")[0]
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[r[ui]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':48s} {'launches':>8s} {'total_us':>11s} {'mean_us':>10s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:48]:48s} {n:8d} {t:11.1f} {t / n:10.2f} {100 * t / tot:6.1f}%")
    lines.append(f"{'TOTAL':48s} {sum(a[0] for a in agg.values()):8d} {tot:11.1f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
