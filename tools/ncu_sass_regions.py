"""Stall breakdown by SASS region of one kernel (tuning aid).
  ncu -i rep --page source --csv --print-source=sass --launch-skip K --launch-count 1 > f.csv
  python tools/ncu_sass_regions.py f.csv [n_regions]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
nreg = int(sys.argv[2]) if len(sys.argv) > 2 else 24
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = {h: hdr.index(h) for h in cols}
isrc = hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iall] or 0) for r in data)
tot_by = {h: sum(int(r[ci[h]] or 0) for r in data) for h in cols}
print("total samples", tot, {k[6:]: v for k, v in sorted(tot_by.items(), key=lambda x: -x[1]) if v})
step = max(1, len(data) // nreg)
for b in range(0, len(data), step):
    seg = data[b:b + step]
    s = sum(int(r[iall] or 0) for r in seg)
    if not s:
        continue
    by = {h[6:]: sum(int(r[ci[h]] or 0) for r in seg) for h in cols}
    top = sorted(by.items(), key=lambda x: -x[1])[:4]
    print(f"{b:5d} {100 * s / tot:5.1f}%  " + " ".join(f"{k}={100 * v / tot:.1f}" for k, v in top if v)
          + f"   | {seg[0][isrc].strip()[:40]}")
