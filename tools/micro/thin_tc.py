"""Time the thin tcgen05 Beaver kernel (mpx_beaver_tc_thin) against the SIMT
tall kernel (mpx_beaver_gemm_sim) at LeNet's conv1 forward shape.
    python tools/micro/thin_tc.py [--reps 20] [--only-thin]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import kernels as Kn  # noqa: E402


def ev(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--only-thin", action="store_true")
ap.add_argument("--shape", default="73728,25,20")
a = ap.parse_args()
L = 3
M, K, N = (int(v) for v in a.shape.split(","))
g = torch.Generator(device="cuda").manual_seed(1)
rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
X, A, C, Y, B = rnd(L, M, K), rnd(L, M, K), rnd(L, M, N), rnd(L, K, N), rnd(L, K, N)
Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
thin = lambda: Kn.beaver_tc_thin(Z, M * N, C.data_ptr(), M * N, X.data_ptr(), M * K, K, 1, A.data_ptr(), M * K,  # noqa
                                 Y.data_ptr(), K * N, N, 1, B.data_ptr(), K * N, L, M, K, N, 0, 64)
t = ev(thin, a.reps)
byts = 8 * L * (2 * M * K + 2 * M * N)
print(f"thin tc: {t:.1f} us, {byts / t / 1e3:.0f} GB/s of X, A, C, Z")
if not a.only_thin:
    Z2 = torch.empty_like(Z)
    simt = lambda: Kn.beaver_gemm_sim(Z2, M * N, L * M * N, C.data_ptr(), M * N, 0, X.data_ptr(), M * K, K, 1, 0,  # noqa
                                      A.data_ptr(), M * K, 0, Y.data_ptr(), K * N, N, 1, 0, B.data_ptr(), K * N, 0,
                                      L, 1, M, K, N, 0, 64)
    t2 = ev(simt, a.reps)
    print(f"simt: {t2:.1f} us; equal: {bool(torch.equal(Z, Z2))}")
