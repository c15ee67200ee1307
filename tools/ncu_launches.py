"""Summarise an ncu --csv launch list that has gpu__time_duration.sum and (optionally)
dram__bytes_read.sum / dram__bytes_write.sum: per kernel launches, mean ms, MB, TB/s.

    python tools/ncu_launches.py launches.csv
"""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID") + 1
    hdr = rows[start - 1]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v = v / 1e6 if u == "ns" else (v / 1e3 if u == "us" else (v * 1e3 if u == "s" else v))
            cnt[name] += 1
        else:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        agg[name][r[mi]] += v
    tot = sum(d["gpu__time_duration.sum"] for d in agg.values())
    lines = [f"{'kernel':28s} {'n':>4s} {'ms/launch':>10s} {'share':>6s} {'MB/launch':>10s} {'TB/s':>6s}"]
    for k, d in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        n = cnt[k]
        t = d["gpu__time_duration.sum"] / n
        by = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / n
        lines.append(f"{k:28s} {n:4d} {t:10.4f} {100 * d['gpu__time_duration.sum'] / tot:5.1f}% {by / 1e6:10.1f} "
                     f"{by / (t / 1e3) / 1e12 if t > 0 else 0:6.2f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
