"""Write a markdown summary of ncu captures (.ncu-rep) and launch lists for profiles/.

    python tools/profile_report.py out.md capture1.ncu-rep [capture2.ncu-rep ...] [--launches launches.csv]
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_static", "static smem/block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def sass_top(rep, n=12):
    """Per kernel section of the source page: top SASS lines by warp-stall samples."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    sections, cur = [], None
    for i, r in enumerate(rows):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1] if len(r) > 1 else "", "hdr": None, "data": []}
            sections.append(cur)
        elif cur is not None and cur["hdr"] is None:
            cur["hdr"] = r
        elif cur is not None:
            cur["data"].append(r)
    res = []
    key = "Warp Stall Sampling (All Samples)"
    for sec in sections:
        h = sec["hdr"] or []
        if key not in h or "Instructions Executed" not in h:
            continue
        ix = {k: i for i, k in enumerate(h)}
        data = [r for r in sec["data"] if len(r) > ix["Instructions Executed"] and r[ix[key]].isdigit()]
        tot = sum(int(r[ix[key]]) for r in data) or 1
        top = sorted(data, key=lambda r: -int(r[ix[key]]))[:n]
        res.append((sec["name"], [(100.0 * int(r[ix[key]]) / tot, int(r[ix["Instructions Executed"]] or 0),
                                   r[ix["Source"]].strip()) for r in top],
                    sum(int(r[ix["Instructions Executed"]] or 0) for r in data)))
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    return tot, cnt


def main():
    out = sys.argv[1]
    args = sys.argv[2:]
    lpath = None
    if "--launches" in args:
        i = args.index("--launches")
        lpath = args[i + 1]
        args = args[:i] + args[i + 2:]
    lines = []
    for rep in args:
        h, units, vals = raw(rep)
        for v in vals:
            name = v[h.index("Kernel Name")]
            lines.append("## %s\n\n`%s`\n" % (name, rep.split("/")[-1]))
            lines.append("| metric | value |\n|---|---|")
            for m, label in METRICS:
                if m in h:
                    lines.append("| %s (`%s`) | %s %s |" % (label, m, v[h.index(m)], units[h.index(m)]))
            lines.append("")
        for kname, top, ninstr in sass_top(rep):
            lines.append("Top SASS lines of `%s` by warp-stall samples (share of samples, warp-level "
                         "executions); %d warp instructions in total:\n" % (kname, ninstr))
            lines.append("```")
            for pct, ex, src in top:
                lines.append("%5.1f%% %12d  %s" % (pct, ex, src))
            lines.append("```\n")
    if lpath:
        tot, cnt = launches(lpath)
        s = sum(tot.values()) or 1
        lines.append("## Launch list `%s` (ncu gpu__time_duration.sum, cold-cache, serialised)\n" % lpath.split("/")[-1])
        lines.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            lines.append("| `%s` | %d | %.3f | %.1f%% |" % (k, cnt[k], v / 1e6, 100 * v / s))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
