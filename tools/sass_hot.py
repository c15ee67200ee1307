"""Hot SASS instructions of an ncu source page (--page source --csv --print-source sass).

    python tools/sass_hot.py source_sass.csv [N]
Prints the N instructions with the most warp-stall samples (and their top stall reasons),
and the local-memory instructions with their execution counts.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"{len(data)} instructions, {tot} samples")
hot = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]
for r in hot:
    smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{r[0][-5:]} {smp:7d} {100 * smp / tot:5.1f}%  exec {r[ix['Instructions Executed']]:>10}  "
          f"{r[1].strip()[:60]:60s} " + " ".join(f"{k}={v}" for v, k in top if v))
print("local memory:")
for r in data:
    if "LDL" in r[1] or "STL" in r[1]:
        print(f"  {r[0][-5:]} exec {r[ix['Instructions Executed']]:>10}  {r[1].strip()}")
