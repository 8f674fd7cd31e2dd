"""Host-side cost of one batch-1 step (cfg3): wall time of the rc_assemble and rc_selective_prefill
calls (host work + launch enqueue, no sync) next to the device time of the step, and the device idle
gap between the step's start event and its first kernel. python profiles/host_overhead.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import rcgen  # noqa: E402


def main():
    wl = rcgen.WORKLOADS["cfg3-llama-4k"]
    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    from paper_2605_07443_b200.build import build
    build()
    env = bench.build_ours(wl, 1, 2, 0, device)
    ctx, lays = env["ctx"], env["batches"][0]
    stream = torch.cuda.current_stream(device)
    n_cand = sum(len(l["cand_idtok"]) for l in lays)
    out = None
    rows = []
    for it in range(25):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t0 = time.perf_counter()
        seqs = ctx.assemble(lays, prefix_id=1, gather_from=1, stream=stream)
        t1 = time.perf_counter()
        out = ctx.selective_prefill(seqs, wl.r_bp, wl.r_bp, check_layer=1, sel_pos=False, hidden=False,
                                    n_cand=n_cand, out=out, stream=stream)
        t2 = time.perf_counter()
        b.record(stream)
        torch.cuda.synchronize()
        ctx.release(seqs)
        if it >= 5:
            rows.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), a.elapsed_time(b)))
    r = np.array(rows)
    med = np.median(r, axis=0)
    print(f"assemble host {med[0]:.3f} ms, prefill host (enqueue) {med[1]:.3f} ms, device step {med[2]:.3f} ms")


if __name__ == "__main__":
    main()
