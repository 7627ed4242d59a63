"""Summarises an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel launches, total and mean device time, share of the total."""
import collections
import csv
import sys


TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarise(path, steps=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
    idi = h.index("ID")
    per = collections.OrderedDict()  # launch id -> (name, {metric: value})
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        v = float(r[vi].replace(",", ""))
        unit, metric = r[ui], r[mi]
        if metric == "gpu__time_duration.sum":
            v *= TIME[unit]
        elif unit in BYTES:
            v *= BYTES[unit]
        per.setdefault(r[idi], (name, {}))[1][metric] = v
    agg = collections.OrderedDict()
    for name, m in per.values():
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    has_bytes = any(a[2] > 0 for a in agg.values())
    hdr = f"{'kernel':44s} {'launches':>8s} {'total_us':>11s} {'mean_us':>10s} {'share':>7s}"
    if has_bytes:
        hdr += f" {'dram_MB/launch':>14s} {'GB/s':>8s}"
    lines = [hdr]
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        line = f"{k[:44]:44s} {n:8d} {t:11.1f} {t / n:10.2f} {100 * t / tot:6.1f}%"
        if has_bytes:
            line += f" {b / n / 1e6:14.1f} {b / (t * 1e3) if t else 0:8.0f}"
        lines.append(line)
    lines.append(f"{'TOTAL':44s} {sum(a[0] for a in agg.values()):8d} {tot:11.1f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
