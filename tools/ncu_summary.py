"""Summarise ncu captures for profiles/ (run here, on the CPU box, on gpurun_out/ files).

    python tools/ncu_summary.py report.ncu-rep [--out profiles/rN/x.txt]
    python tools/ncu_summary.py launches.csv            # a --metrics gpu__time_duration.sum list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__warps_active.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sass__inst_executed_local_loads",
    "sass__inst_executed_local_stores",
]
STALLS = "smsp__average_warps_issue_stalled_"


def summarize_rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        out.append(f"== {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:75s} {d[k]:>20s} {u.get(k, '')}")
        st = sorted(((float(d[k] or 0), k) for k in d if k.startswith(STALLS) and k.endswith("per_issue_active.ratio")),
                    reverse=True)[:8]
        out.append("  top stall reasons (warps per issue):")
        for v, k in st:
            out.append(f"    {k[len(STALLS):]:60s} {v:8.3f}")
    return "\n".join(out)


def summarize_csv(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'ms':>12s} {'launches':>8s} {'share':>6s}  kernel (ncu serialised, cold-cache: compare shares)"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t:12.3f} {n:8d} {100 * t / tot:5.1f}%  {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    p = sys.argv[1]
    txt = summarize_rep(p) if p.endswith(".ncu-rep") else summarize_csv(p)
    if "--out" in sys.argv:
        open(sys.argv[sys.argv.index("--out") + 1], "w").write(txt + "\n")
    print(txt)
