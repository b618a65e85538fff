"""Sim-mode Beaver product at one shape: fused mask+limb (mpx_mask_limbs2) and
the split-operand tcgen05 GEMM (mpx_gemm_limbs_split), timed separately with
CUDA events; checks the GEMM against the u64 SIMT reconstruction.

    python tools/micro/gemm_split_shapes.py [--only m,k,r] [--parties 3] [--reps 20]
Default shapes: the LeNet batch-128 step's tcgen05 products.  MPX_TC_* env
knobs (MPX_TC_KSPLIT ...) apply.  For ncu: --reps 1 and -k regex:k_gemm_limbs.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import kernels as K  # noqa: E402

LENET_TC = [(8192, 500, 50), (128, 800, 500), (800, 128, 500), (128, 500, 800), (500, 8192, 50), (8192, 50, 500)]


def ev_time(fn, reps):
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


def run(m, k, r, L, reps, check):
    g = torch.Generator(device="cuda").manual_seed(1)
    rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
    X, A, C = rnd(L, m, k), rnd(L, m, k), rnd(L, m, r)
    Y, B = rnd(L, k, r), rnd(L, k, r)
    Z = torch.empty((L, m, r), dtype=torch.int64, device="cuda")
    Mp, Np, Kh = K._rup(m, 128), K._rup(r, 32), K.kpad(k)
    SA = torch.empty((8, Mp, Kh), dtype=torch.uint8, device="cuda")
    PA = torch.empty((L, 8, Mp, Kh), dtype=torch.uint8, device="cuda")
    SB = torch.empty((8, Np, Kh), dtype=torch.uint8, device="cuda")
    PB = torch.empty((L, 8, Np, Kh), dtype=torch.uint8, device="cuda")

    def mask():
        K.mask_limbs2(SA, PA, X.data_ptr(), m * k, k, 1, A.data_ptr(), m * k, k, 1, m, Mp,
                      SB, PB, Y.data_ptr(), k * r, 1, r, B.data_ptr(), k * r, 1, r, r, Np, L, k, Kh, 0, 64)

    def gemm():
        K.gemm_limbs_split(Z, PA, SA, PB, SB, L, m, r, Mp, Np, Kh, r, m * r, 64, C.data_ptr(), m * r)

    mask()
    tm = ev_time(mask, reps)
    tg = ev_time(gemm, reps)
    ok = None
    if check:
        D = (X.sum(0) - A.sum(0))
        E = (Y.sum(0) - B.sum(0))
        Zs = torch.empty_like(Z)
        K.beaver_gemm(Zs, m * r, C.data_ptr(), m * r, D, E, A.data_ptr(), m * k, B.data_ptr(), k * r, L, m, k, r, 0, 64)
        ok = bool(torch.equal(Z, Zs))
    ops = 2 * 36 * L * Mp * K._rup(r, 32) * 2 * Kh
    alg = 2 * 36 * L * m * r * 2 * k
    return {"m": m, "k": k, "r": r, "L": L, "mask_us": round(tm, 1), "gemm_us": round(tg, 1),
            "padded_TOPS": round(ops / tg / 1e6, 1), "alg_TOPS": round(alg / tg / 1e6, 1), "exact": ok}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--parties", type=int, default=3)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-check", action="store_true")
    a = ap.parse_args()
    shapes = [tuple(int(v) for v in a.only.split(","))] if a.only else LENET_TC
    tot = 0.0
    for m, k, r in shapes:
        res = run(m, k, r, a.parties, a.reps, not a.no_check)
        tot += res["gemm_us"]
        print(json.dumps(res), flush=True)
    print(json.dumps({"gemm_total_us": round(tot, 1)}))


if __name__ == "__main__":
    main()
