"""Time the tcgen05 limb GEMM kernel alone (split excluded / included).

    python tools/bench_gemm.py [--m 4096 --n 4096 --k 8192] [--iters 10]

Reports int8 limb TOPS (36 u8 MACs per ring MAC, 2 ops per MAC) and the
ring-GMAC/s rate, CUDA-event timed after warm-up.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_02320_b200 import kernels as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    M, N, Kd, b = a.m, a.n, a.k, a.batch
    Mpad, Npad, Kpad = (M + 127) // 128 * 128, (N + 63) // 64 * 64, (Kd + 127) // 128 * 128
    A8 = torch.randint(0, 256, (b, 8, Mpad, Kpad), dtype=torch.uint8, device="cuda")
    B8 = torch.randint(0, 256, (b, 8, Npad, Kpad), dtype=torch.uint8, device="cuda")
    C = torch.zeros((b, M, N), dtype=torch.int64, device="cuda")
    A = torch.randint(-(1 << 62), 1 << 62, (M, Kd), dtype=torch.int64, device="cuda")
    B = torch.randint(-(1 << 62), 1 << 62, (Kd, N), dtype=torch.int64, device="cuda")
    for _ in range(3):
        K.gemm_limbs(C, A8, B8, b, M, N, Mpad, Npad, Kpad, N, M * N, False, 64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        K.gemm_limbs(C, A8, B8, b, M, N, Mpad, Npad, Kpad, N, M * N, False, 64)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    macs = b * M * N * Kd
    # full u64 path incl. splits
    for _ in range(2):
        K.gemm_tc(C[0], A, B, 1, M, Kd, N, 0, 0, 0, False, 64)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        K.gemm_tc(C[0], A, B, 1, M, Kd, N, 0, 0, 0, False, 64)
    e1.record()
    torch.cuda.synchronize()
    ms_full = e0.elapsed_time(e1) / a.iters
    print(json.dumps({"M": M, "N": N, "K": Kd, "batch": b, "kernel_ms": ms,
                      "int8_TOPS": 36 * 2 * macs / ms / 1e9, "ring_GMACs": macs / ms / 1e6,
                      "full_u64_ms_batch1": ms_full, "full_int8_TOPS": 36 * 2 * M * N * Kd / ms_full / 1e9}))


if __name__ == "__main__":
    main()
