"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes + tensor-pipe activity per
launch) of `bench.py --profile-only --steps 1 --warmup 1` into a per-kernel table for the LAST step
(the profiled step). python profiles/launch_table.py <launches.csv> [gemm_traffic_json]"""
import collections
import csv
import json
import re
import sys


def main(path, traffic_out=None):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h, rows = rows[0], rows[1:]
    ID, K, MN, MV = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    by = collections.OrderedDict()
    for r in rows:
        d = by.setdefault(r[ID], {"name": r[K]})
        d[r[MN]] = float(r[MV].replace(",", ""))
    ks = list(by.values())

    def short(n):
        m = re.search(r"(k_\w+)(<[^>]*>)?", n)
        return (m.group(1) + (m.group(2) or "")).replace("(int)", "") if m else n[:30]
    emb = [i for i, x in enumerate(ks) if "k_embed" in x["name"]]
    last = ks[emb[-1]:]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for x in last:
        a = agg[short(x["name"])]
        t = x["gpu__time_duration.sum"]
        a[0] += 1
        a[1] += t
        a[2] += x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
        a[3] += x.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0) * t
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':24s} {'launches':>8s} {'ms/step':>9s} {'share':>6s} {'DRAM MB/launch':>15s} {'tensor active':>13s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:24s} {a[0]:8d} {a[1] / 1e6:9.3f} {a[1] / tot:6.3f} {a[2] / a[0] / 1e6:15.1f} {a[3] / a[1]:12.1f}%")
    print(f"{'total':24s} {'':8s} {tot / 1e6:9.3f}")
    if traffic_out:
        g = [x for x in last if "k_gemm" in x["name"]]
        b = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in g) / len(g)
        json.dump({"gemm_bytes_per_launch": b, "launches": len(g),
                   "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum, mean over the {len(g)} GEMM launches "
                             f"of one cfg3 batch-32 step ({path})"}, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
