"""Summarise one-kernel ncu reports: key raw metrics, stall samples, and the source lines with the
most executed instructions. usage: python tools/ncu_summary.py report.ncu-rep [n_lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nlines = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[-1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
for i, n in enumerate(h):
    if n in want:
        print("%-60s %s %s" % (n, v[i], rows[1][i]))
st = [(h[i], float(v[i] or 0)) for i in range(len(h))
      if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")]
tot = sum(x for _, x in st) or 1
print("stalls:", ", ".join("%s %.1f%%" % (n.replace("smsp__pcsamp_warps_issue_stalled_", ""), 100 * x / tot)
                           for n, x in sorted(st, key=lambda a: -a[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
cur, agg = None, {}
for r in rows[hi + 1:]:
    if r and r[0] and r[0].isdigit():
        cur = (int(r[0]), r[1].strip()[:90])
        agg.setdefault(cur, [0.0, 0.0])
        continue
    if cur is None or len(r) <= ie:
        continue
    try:
        agg[cur][0] += float(r[ie] or 0)
        agg[cur][1] += float(r[ss] or 0)
    except ValueError:
        pass
T = sum(a[0] for a in agg.values()) or 1
S = sum(a[1] for a in agg.values()) or 1
print("instructions %.3e" % T)
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:nlines]:
    print("%5.1f%% inst %5.1f%% stall  L%d %s" % (100 * a[0] / T, 100 * a[1] / S, key[0], key[1]))
