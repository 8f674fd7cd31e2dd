"""Micro-benchmark of the tcgen05 GEMM kernels in isolation (rc_diag_gemm, EPI_F32 epilogue) over
small-M shapes: us per launch and TFLOP/s with the weight operand hot in L2 (one B reused) or cold
(rotating over enough copies to exceed the 126 MB L2). Run once per env setting, e.g.
RC_GEMM_PAIR_MIN_M=512 python profiles/micro/gemm_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2605_07443_b200.api import diag_gemm  # noqa: E402


def run(M, N, K, cold, reps=12):
    dev = torch.device("cuda", 0)
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    wbytes = N * K * 2
    ncopy = max(1, -(-300 * 2**20 // wbytes)) if cold else 1
    Bs = [torch.randn(N, K, device=dev).to(torch.bfloat16) for _ in range(ncopy)]
    for i in range(3):
        diag_gemm(A, Bs[i % ncopy])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        diag_gemm(A, Bs[i % ncopy])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    return us, 2.0 * M * N * K / us / 1e6


if __name__ == "__main__":
    tag = os.environ.get("TAG", "default")
    shapes = [(625, 28672, 4096), (625, 6144, 4096), (625, 4096, 14336), (1250, 28672, 4096), (2500, 28672, 4096),
              (5000, 28672, 4096), (640, 28672, 4096), (512, 28672, 4096), (768, 28672, 4096)]
    for (M, N, K) in shapes:
        for cold in (False, True):
            us, tf = run(M, N, K, cold)
            print(f"{tag:10s} M={M:5d} N={N:5d} K={K:5d} {'cold' if cold else 'hot ':4s} {us:8.1f} us {tf:7.1f} TFLOP/s",
                  flush=True)
