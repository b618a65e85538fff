"""Time mpx_beaver_gemm_sim (fused sim-mode Beaver product) vs the
mask + mask + mpx_beaver_gemm_batched sequence on given shapes.

    python tools/micro/bs_sweep.py [--parties 3]
"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import kernels as K  # noqa: E402

SHAPES = [(73728, 25, 20, False, False), (25, 73728, 20, True, False), (128, 500, 10, False, False), (500, 128, 10, True, False),
          (128, 10, 500, False, True), (27, 131072, 64, True, False)]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parties", type=int, default=3)
    L = ap.parse_args().parties
    g = torch.Generator(device="cuda").manual_seed(1)
    rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
    for m, k, r, xt, yt in SHAPES:
        X = rnd(L, k, m).transpose(1, 2) if xt else rnd(L, m, k)
        Y = rnd(L, r, k).transpose(1, 2) if yt else rnd(L, k, r)
        A, B, C = rnd(L, m, k), rnd(L, k, r), rnd(L, m, r)
        Z = torch.empty((L, m, r), dtype=torch.int64, device="cuda")
        t = timeit(lambda: K.beaver_gemm_sim(Z, m * r, 0, C.data_ptr(), m * r, 0, X.data_ptr(), X.stride(0),
                                             X.stride(1), X.stride(2), 0, A.data_ptr(), m * k, 0, Y.data_ptr(),
                                             Y.stride(0), Y.stride(1), Y.stride(2), 0, B.data_ptr(), k * r, 0, L, 1,
                                             m, k, r, 0, 64))
        D, E = rnd(m, k), rnd(k, r)
        tg = timeit(lambda: K.beaver_gemm(Z, m * r, C.data_ptr(), m * r, D, E, A.data_ptr(), m * k, B.data_ptr(),
                                          k * r, L, m, k, r, 0, 64))
        macs = 2 * L * m * k * r
        print(f"{m}x{k}x{r} L={L} per_sm={os.environ.get('MPX_BS_PER_SM', '-')}: sim {t:.1f} us "
              f"({macs / t / 1e6:.2f} T u64-MAC/s)  gemm-only {tg:.1f} us", flush=True)


if __name__ == "__main__":
    main()
