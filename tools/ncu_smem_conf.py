"""Per-SASS shared-memory wavefronts vs ideal from an ncu report (bank-conflict hot spots)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
print("columns:", [h for h in hh if "hared" in h or "Conflict" in h or "Wavefront" in h])
ia, isrc, ie = hh.index("Address"), hh.index("Source"), hh.index("Instructions Executed")
cols = [i for i, h in enumerate(hh) if "hared" in h or "Conflict" in h or "Wavefront" in h]
out = []
for r in rows[2:]:
    if len(r) < len(hh):
        continue
    vals = []
    for i in cols:
        try:
            vals.append(float(r[i] or 0))
        except ValueError:
            vals.append(0.0)
    if any(vals):
        out.append((vals, r[ia], r[isrc].strip()[:70], r[ie]))
out.sort(key=lambda x: -max(x[0]))
for vals, a, s, n in out[:60]:
    print(a, n, " ".join(f"{v:.0f}" for v in vals), s)
