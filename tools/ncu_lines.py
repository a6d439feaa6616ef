"""Per-CUDA-line instruction/stall attribution from an ncu report (mixed source+SASS view)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname = None; hdr = None; cur_line = None; cur_src = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None:
        continue
    if r[0]:  # a CUDA source line row
        cur_line, cur_src = r[0], r[1]
    ie = hdr.index("Instructions Executed"); iss = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        n = float(r[ie] or 0); s = float(r[iss] or 0)
    except (ValueError, IndexError):
        continue
    if not r[0] and r[2]:  # SASS row under the current CUDA line
        key = (fname, cur_line)
        a = agg.setdefault(key, [0.0, 0.0, cur_src])
        a[0] += n; a[1] += s
tot = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print(f"total warp instructions {tot:.4g}")
for (f, l), (n, s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*n/tot:5.1f}% inst {100*s/max(ts,1):5.1f}% stall  {f}:{l}  {src.strip()[:90]}")
print("-- by stall samples")
for (f, l), (n, s, src) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*n/tot:5.1f}% inst {100*s/max(ts,1):5.1f}% stall  {f}:{l}  {src.strip()[:90]}")
