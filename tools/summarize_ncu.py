"""Summarise ncu captures into profiles/ (run in the build container).

    python tools/summarize_ncu.py <tag> <report.ncu-rep>...   -> profiles/<tag>_ncu_summary.json/.md
    python tools/summarize_ncu.py --launches <tag> <launches.csv>

The .ncu-rep files themselves stay in gpurun_out/ (scratch); the summaries are
what is committed.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_membar",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_requests_srcunit_tex.sum",
]


def raw(rep):
    # a .ncu-rep, or the `ncu -i ... --page raw --csv` text of one (.csv)
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 10]
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:90]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = {}
    order = []
    for r in rows[1:]:
        k = r[ki].split("(")[0].replace("void ", "")
        if k not in per:
            order.append(k)
            per[k] = [0, 0.0]
        per[k][0] += 1
        per[k][1] += float(r[vi].replace(",", "")) / 1000.0
    return [{"kernel": k, "launches": per[k][0], "total_us": round(per[k][1], 1)} for k in order]


def main():
    args = sys.argv[1:]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if args[0] == "--launches":
        tag, path = args[1], args[2]
        res = launches(path)
        tot = sum(r["total_us"] for r in res)
        for r in res:
            r["share"] = round(r["total_us"] / tot, 4) if tot else 0
        out = os.path.join(ROOT, "profiles", f"{tag}_launches.json")
        json.dump({"source": os.path.basename(path), "kernels": res, "total_us": round(tot, 1)},
                  open(out, "w"), indent=1)
        print(out)
        return
    tag, reps = args[0], args[1:]
    allres = {}
    for rep in reps:
        allres[os.path.basename(rep)] = raw(rep)
    out = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.json")
    json.dump(allres, open(out, "w"), indent=1)
    md = [f"# ncu summaries ({tag})", ""]
    for rep, res in allres.items():
        for d in res:
            md.append(f"## {rep}: {d['kernel']}")
            for m in METRICS:
                if m in d:
                    md.append(f"- {m}: {d[m]}")
            md.append("")
    open(out.replace(".json", ".md"), "w").write("\n".join(md))
    print(out)


if __name__ == "__main__":
    main()
