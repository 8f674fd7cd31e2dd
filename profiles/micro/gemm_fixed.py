"""Fixed vs per-k-block cost of the tcgen05 GEMM at batch-1 shapes: one-round launches (M = 625,
N = 6144: 120 single-CTA tiles) over K = 512 .. 8192, plus a one-tile launch; the intercept of us vs K
is the launch's fixed cost (prologue, pipeline fill, epilogue, teardown), the slope the k-block rate."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2605_07443_b200.api import diag_gemm  # noqa: E402


def run(M, N, K, reps=20):
    dev = torch.device("cuda", 0)
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    B = torch.randn(N, K, device=dev).to(torch.bfloat16)
    for _ in range(3):
        diag_gemm(A, B)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        diag_gemm(A, B)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


if __name__ == "__main__":
    tag = os.environ.get("TAG", "default")
    for (M, N) in [(625, 6144), (128, 256), (128, 256 * 148), (256, 256 * 74)]:
        for K in (512, 1024, 2048, 4096, 8192):
            us = run(M, N, K)
            print(f"{tag:8s} M={M:5d} N={N:6d} K={K:5d} {us:8.2f} us  {2.0 * M * N * K / us / 1e6:7.1f} TFLOP/s", flush=True)
