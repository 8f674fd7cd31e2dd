"""Format the sweep_*.json bench lines of profiles/sweep.sh into the r01_sweep.txt table.
python profiles/sweep_table.py <dir with sweep_*.json>"""
import glob
import json
import os
import sys


def main(d):
    rows = []
    for f in sorted(glob.glob(os.path.join(d, "sweep_*.json"))):
        txt = open(f).read().strip().splitlines()
        if not txt:
            continue
        x = json.loads(txt[-1])
        c, k, b = x["config"], x.get("kernels", {}), x.get("baselines") or {}
        base = ""
        if b:
            t = b.get("ttft_b1_ms", {})
            base = (f"full ours {t.get('full_ours_p50', 0):.1f} ms, torch {t.get('full_torch_p50', 0):.1f} ms, "
                    f"prefix-cache {t.get('prefix_cache_ours_p50', 0):.1f} ms; "
                    f"ttft_b1_speedup_vs_full={b.get('ttft_b1_speedup_vs_full', 0):.2f}")
        rows.append((c["workload"], c["batch"], c["r"], x["value"], x["ms_per_step"], x["ttft_ms"]["p50"],
                     x["ttft_ms"]["p99"], k.get("gemm", {}).get("tflops", 0), k.get("gemm", {}).get("frac_tensor", 0),
                     k.get("attention", {}).get("ms_per_step", 0), x["clocks"]["sm_mhz"], base))
    rows.sort(key=lambda r: (r[0], r[1], r[2]))
    print("SURVEY §8(d) sweep (profiles/sweep.sh), one B200, bench.py JSON lines; TTFT = device time per batch")
    print(f"{'config':14s} {'batch':>5s} {'r':>5s} {'tok/s':>9s} {'ms/step':>8s} {'TTFT p50':>9s} {'p99':>8s} "
          f"{'GEMM TF/s':>9s} {'frac':>5s} {'attn ms':>8s} {'sm MHz':>7s}  baselines")
    for r in rows:
        print(f"{r[0]:14s} {r[1]:5d} {r[2]:5.2f} {r[3]:9.0f} {r[4]:8.2f} {r[5]:9.2f} {r[6]:8.2f} {r[7]:9.0f} "
              f"{r[8]:5.2f} {r[9]:8.2f} {str(r[10]):>7s}  {r[11]}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
