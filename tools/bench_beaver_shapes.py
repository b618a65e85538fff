"""Time the Beaver matrix-product reconstruction per shape on both kernels:
SIMT one-launch (mpx_beaver_gemm) vs tcgen05 limbs (beaver_limbs + gemm_limbs).

    python tools/bench_beaver_shapes.py [--parties 3]
Shapes default to the LeNet batch-128 training step's products (m, k, r).
"""
import argparse, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_02320_b200 import kernels as K  # noqa: E402

LENET = [(73728, 25, 20), (25, 73728, 20), (8192, 500, 50), (500, 8192, 50), (8192, 50, 500),
         (128, 800, 500), (800, 128, 500), (128, 500, 800), (128, 500, 10), (500, 128, 10), (128, 10, 500)]


def _vgg():
    convs = [(3, 64, 32), (64, 64, 32), (64, 128, 16), (128, 128, 16), (128, 256, 8), (256, 256, 8),
             (256, 512, 4), (512, 512, 4), (512, 512, 2)]
    out = []
    for cin, cout, hw in convs:
        m, k = 128 * hw * hw, 9 * cin
        out += [(m, k, cout), (k, m, cout), (m, cout, k)]      # forward, dW, dX
    return out


REPS = [20]


def timeit(fn, reps=None):
    reps = reps or REPS[0]
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


def _tc_time(m, k, r, L):
    """GEMM-only time (limb planes prepared once) of the Beaver product."""
    g = torch.Generator(device="cuda").manual_seed(1)
    rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
    D, E = rnd(m, k), rnd(k, r)
    A, B, C = rnd(L, m, k), rnd(L, k, r), rnd(L, m, r)
    Z = torch.empty((L, m, r), dtype=torch.int64, device="cuda")
    Mp, Np, Kp = K._rup(m, 128), K._rup(r, 32), K.kpad(2 * k)
    A8 = torch.zeros((L, 8, Mp, Kp), dtype=torch.uint8, device="cuda")
    B8 = torch.empty((L, 8, Np, Kp), dtype=torch.uint8, device="cuda")
    K.beaver_limbs(A8, B8, D, E, A.data_ptr(), m * k, B.data_ptr(), k * r, L, m, k, r, Mp, Np, Kp, 0)
    return timeit(lambda: K.gemm_limbs(Z, A8, B8, L, m, r, Mp, Np, Kp, r, m * r, False, 64, cin=C, s_cin=m * r))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parties", type=int, default=3)
    ap.add_argument("--shapes", default="lenet")
    ap.add_argument("--no-simt", action="store_true")
    ap.add_argument("--only", default=None, help="m,k,r")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--splits", default=None, help="comma list of forced split-K counts")
    a = ap.parse_args()
    L = a.parties
    REPS[0] = a.reps
    out = []
    shapes = _vgg() if a.shapes == "vgg" else LENET
    if a.only:
        shapes = [tuple(int(v) for v in a.only.split(","))]
    if a.splits:
        for m, k, r in shapes:
            res = {}
            for sp in a.splits.split(","):
                os.environ["MPX_TC_KSPLIT"] = sp
                res[sp] = round(_tc_time(m, k, r, L), 1)
            os.environ.pop("MPX_TC_KSPLIT", None)
            res["auto"] = round(_tc_time(m, k, r, L), 1)
            print(json.dumps({"m": m, "k": k, "r": r, "gemm_us_by_split": res}), flush=True)
        return
    for m, k, r in shapes:
        g = torch.Generator(device="cuda").manual_seed(1)
        rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
        D, E = rnd(m, k), rnd(k, r)
        A, B, C = rnd(L, m, k), rnd(L, k, r), rnd(L, m, r)
        Z = torch.empty((L, m, r), dtype=torch.int64, device="cuda")
        simt = None if a.no_simt else timeit(
            lambda: K.beaver_gemm(Z, m * r, C.data_ptr(), m * r, D, E, A.data_ptr(), m * k, B.data_ptr(),
                                  k * r, L, m, k, r, 0, 64))
        Zs = Z.clone()
        Mp, Np, Kp = K._rup(m, 128), K._rup(r, 32), K.kpad(2 * k)
        A8 = torch.zeros((L, 8, Mp, Kp), dtype=torch.uint8, device="cuda")
        B8 = torch.empty((L, 8, Np, Kp), dtype=torch.uint8, device="cuda")

        def tc():
            K.beaver_limbs(A8, B8, D, E, A.data_ptr(), m * k, B.data_ptr(), k * r, L, m, k, r, Mp, Np, Kp, 0)
            K.gemm_limbs(Z, A8, B8, L, m, r, Mp, Np, Kp, r, m * r, False, 64, cin=C, s_cin=m * r)
        t = timeit(tc)
        same = None if simt is None else bool(torch.equal(Z, Zs))
        lim = timeit(lambda: K.beaver_limbs(A8, B8, D, E, A.data_ptr(), m * k, B.data_ptr(), k * r, L, m, k, r, Mp,
                                            Np, Kp, 0))
        ops = 2 * 36 * L * Mp * Np * Kp
        out.append({"m": m, "k": k, "r": r, "simt_us": None if simt is None else round(simt, 1), "tc_us": round(t, 1),
                    "limbs_us": round(lim, 1), "gemm_TOPS": round(ops / ((t - lim) * 1e-6) / 1e12, 1), "equal": same})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
