"""Print the headline counters of an .ncu-rep (first profiled kernel)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units, v = r[0], r[1], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_read.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]
for k in keys:
    if k in h:
        print(f"{k}: {v[h.index(k)]} {units[h.index(k)]}")
st = [(float(v[i] or 0), h[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
for val, k in sorted(st, reverse=True)[:10]:
    print(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', 'stall_')}: {val:.0f}")
