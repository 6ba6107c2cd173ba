"""Summarise ncu captures into committed markdown (profiles/).

    python tools/summarize_ncu.py report.ncu-rep [...] > profiles/<name>.md
    python tools/summarize_ncu.py --launches launches.csv > profiles/<name>.md
"""
import collections
import csv
import subprocess
import sys

METRICS = [
    ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs/thread"),
    ("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 (LTS) %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, data = rows[0], rows[1], rows[2:]
    stall_cols = [i for i, x in enumerate(h)
                  if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio")]
    print("## `%s`\n" % path.split("/")[-1])
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0]
        print("### %s\n" % name)
        print("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                print("| %s | %s %s |" % (label, r[i], u[i]))
        st = sorted(((float(r[i] or 0), h[i][len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                     for i in stall_cols), reverse=True)[:6]
        print("| top stalls (per issue) | %s |\n" % ", ".join("%s %.2f" % (n, v) for v, n in st))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) > 5]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    print("Kernel launches inside the NVTX range `timed_steps` (one layer step), ncu "
          "`gpu__time_duration.sum` (cold-cache, serialised): %d launches, %.2f ms total.\n" % (len(data), T / 1e6))
    print("| kernel | launches | ms | share | avg us |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print("| %s | %d | %.2f | %.1f%% | %.1f |" % (k.replace("<unnamed>::", ""), cnt[k], v / 1e6, 100 * v / T,
                                                    v / cnt[k] / 1e3))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[1:]:
            report(p)
