"""Dump per-SASS-instruction executed counts of an ncu report: address, opcode, count, stall samples."""
import csv, io, subprocess, sys
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ie, isrc, ia = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Address")
iss = hh.index("Warp Stall Sampling (All Samples)")
for r in rows[2:]:
    if len(r) < len(hh):
        continue
    try:
        n = float(r[ie] or 0); s = float(r[iss] or 0)
    except ValueError:
        continue
    print(f"{r[ia]}\t{int(n)}\t{int(s)}\t{r[isrc].strip()[:80]}")
