"""Summarise an ncu launch list (gpu__time_duration per launch) and ncu --set full reports into
the per-kernel tables committed under profiles/.

  python profiles/ncu_summary.py launches <launches.csv> <n_steps>      # share of each kernel per step
  python profiles/ncu_summary.py full <report.ncu-rep>                  # key counters per profiled launch
"""
import collections
import csv
import re
import subprocess
import sys

SETUP = ("k_pool_transpose", "k_scale_transpose")


def base(name):
    m = re.search(r"(k_\w+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:40]


def launches(path, steps):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        k = base(r[4])
        if k.startswith(SETUP):
            continue
        tot[k] += float(r[-1]) / 1e6  # ns -> ms
        cnt[k] += 1
    s = sum(tot.values())
    print(f"{'kernel':40s} {'ms/step':>9s} {'launch/step':>11s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:40s} {v / steps:9.3f} {cnt[k] / steps:11.1f} {100 * v / s:6.1f}%")
    print(f"{'total':40s} {s / steps:9.3f}")


FULL = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__registers_per_thread"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(base(d["Kernel Name"]))
        for k in FULL:
            if k in d:
                print(f"   {k:70s} {d[k]:>14s} {units[hdr.index(k)]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]))
    else:
        full(sys.argv[2])
