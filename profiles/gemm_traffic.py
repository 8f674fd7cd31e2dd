"""DRAM traffic of every GEMM class in one cfg3 step against its algorithmic bytes and the Hong-Kung
I/O lower bound of a matmul with fast memory S (the 126 MB L2): words moved >= 2 M N K / sqrt(S)
beyond the output writes. python profiles/gemm_traffic.py <launches.csv> <batch>

Classes follow the launch order of a step (rc_api.cu): layer 0 over U (QKV, O, gate/up, down), the
check-layer K/V GEMM (deviation), then per selective layer QKV, O, gate/up, down over the Sel rows."""
import collections
import csv
import math
import sys

D, H, HK, DH, F, L = 4096, 32, 8, 128, 14336, 32
N_TOK, P, SEL = 4096, 207, 625
S_WORDS = 126e6 / 2  # L2 in bf16 words


def shapes(batch):
    U, S = (N_TOK - P) * batch, SEL * batch
    qkv, kvn = (H + 2 * HK) * DH, 2 * HK * DH
    # (M, N, K, output bytes per element)
    return {"layer0 qkv": (U, qkv, D, 2), "layer0 o": (U, D, H * DH, 8), "layer0 gate/up": (U, 2 * F, D, 1),
            "layer0 down": (U, D, F, 8), "check kv (dev)": (U, kvn, D, 0), "sel qkv": (S, qkv, D, 2),
            "sel o": (S, D, H * DH, 8), "sel gate/up": (S, 2 * F, D, 1), "sel down": (S, D, F, 8)}


def bounds(M, N, K, ob):
    alg = 2 * (M * K + N * K) + ob * M * N
    hk = max(alg, 2 * 2 * M * N * K / math.sqrt(S_WORDS) + ob * M * N)
    return alg, hk


def main(path, batch):
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
    emb = [i for i, x in enumerate(ks) if "k_embed" in x["name"]][-1]
    gem = [x for x in ks[emb:] if "k_gemm" in x["name"]]
    order = ["layer0 qkv", "layer0 o", "layer0 gate/up", "layer0 down", "check kv (dev)"]
    order += ["sel qkv", "sel o", "sel gate/up", "sel down"] * (L - 1)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for cls, x in zip(order, gem):
        a = agg[cls]
        a[0] += 1
        a[1] += x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
        a[2] += x.get("gpu__time_duration.sum", 0)
    sh = shapes(batch)
    print(f"# cfg3 batch {batch}: DRAM bytes per launch (ncu, cold L2 per launch) vs algorithmic and vs the "
          f"Hong-Kung bound 2MNK/sqrt(S) (S = 126 MB of L2) + output")
    print(f"{'class':16s} {'launches':>8s} {'M':>7s} {'N':>6s} {'K':>6s} {'alg GB':>8s} {'HK GB':>8s} {'DRAM GB':>8s} "
          f"{'x alg':>6s} {'x HK':>6s}")
    for cls in dict.fromkeys(order):
        if cls not in agg:
            continue
        n, byt, _ = agg[cls]
        M, N, Kd, ob = sh[cls]
        alg, hk = bounds(M, N, Kd, ob)
        got = byt / n
        print(f"{cls:16s} {n:8d} {M:7d} {N:6d} {Kd:6d} {alg / 1e9:8.3f} {hk / 1e9:8.3f} {got / 1e9:8.3f} "
              f"{got / alg:6.2f} {got / hk:6.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
