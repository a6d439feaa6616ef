"""Summarise an ncu report: key metrics + SASS opcode mix + hot address windows."""
import csv, subprocess, sys, io, json
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"]
out = {}
for i, n in enumerate(h):
    if n in keys:
        out[n] = (v[i], u[i])
for k in keys:
    if k in out:
        print(f"{k:80s} {out[k][0]:>16s} {out[k][1]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ie, isrc, ia = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Address")
iss = hh.index("Warp Stall Sampling (All Samples)")
tot = 0; byop = {}; samp = 0; bysamp = {}
for r_ in rows[2:]:
    if len(r_) < len(hh):
        continue
    try:
        n = float(r_[ie] or 0); s = float(r_[iss] or 0)
    except ValueError:
        continue
    parts = r_[isrc].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") else parts[0]
    op = op.split(".")[0]
    tot += n; samp += s
    byop[op] = byop.get(op, 0) + n
    bysamp[op] = bysamp.get(op, 0) + s
print(f"total warp instructions {tot:.4g}")
for k, val in sorted(byop.items(), key=lambda x: -x[1])[:16]:
    print(f"  {k:12s} {100 * val / tot:6.2f}% inst  {100 * bysamp[k] / max(samp, 1):6.2f}% stall-samples")
