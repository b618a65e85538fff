"""Time the long-K tcgen05 Beaver kernel (mpx_beaver_tc_long) against the SIMT
kernel (mpx_beaver_gemm_sim) at LeNet's conv1 weight-gradient shape
(cols^T @ dZ: 25 x 73728 x 20, three parties, X a transposed view), plus the
MPX_LONG_DBG skeleton variants (1 no loads, 2 no conversion, 4 no MMA).
    python tools/micro/long_tc.py [--reps 20] [--shape M,K,N]"""
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
ap.add_argument("--shape", default="25,73728,20")
a = ap.parse_args()
L = 3
M, K, N = (int(v) for v in a.shape.split(","))
g = torch.Generator(device="cuda").manual_seed(1)
rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
XT, A, C, Y, B = rnd(L, K, M), rnd(L, M, K), rnd(L, M, N), rnd(L, K, N), rnd(L, K, N)
Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
lng = lambda: Kn.beaver_tc_long(Z, M * N, C.data_ptr(), M * N, XT.data_ptr(), K * M, 1, M, A.data_ptr(), M * K,  # noqa
                                Y.data_ptr(), K * N, N, 1, B.data_ptr(), K * N, L, M, K, N, 0, 64)
byts = 8 * L * (2 * M * K + 2 * K * N)
t = ev(lng, a.reps)
print(f"long tc: {t:.1f} us, {byts / t / 1e3:.0f} GB/s of X, A, Y, B")
for dbg in ((1, 2, 4, 3, 5, 6, 7) if "MPX_LONG_DBG" not in os.environ and a.reps > 1 else ()):
    os.environ["MPX_LONG_DBG"] = str(dbg)
    print(f"  dbg {dbg}: {ev(lng, a.reps):.1f} us")
os.environ.pop("MPX_LONG_DBG", None)
Z2 = torch.empty_like(Z)
simt = lambda: Kn.beaver_gemm_sim(Z2, M * N, L * M * N, C.data_ptr(), M * N, 0, XT.data_ptr(), K * M, 1, M, 0,  # noqa
                                  A.data_ptr(), M * K, 0, Y.data_ptr(), K * N, N, 1, 0, B.data_ptr(), K * N, 0,
                                  L, 1, M, K, N, 0, 64)
t2 = ev(simt, a.reps)
lng()
print(f"simt: {t2:.1f} us; equal: {bool(torch.equal(Z, Z2))}")
