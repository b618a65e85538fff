"""One shape of mpx_beaver_gemm_sim (for ncu): python tools/micro/bs_one.py m k r [L] [xt]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import kernels as K  # noqa: E402

m, k, r = (int(a) for a in sys.argv[1:4])
L = int(sys.argv[4]) if len(sys.argv) > 4 else 3
xt = len(sys.argv) <= 5 or sys.argv[5] == "1"
g = torch.Generator(device="cuda").manual_seed(1)
rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
X = rnd(L, k, m).transpose(1, 2) if xt else rnd(L, m, k)
Y, A, B, C = rnd(L, k, r), rnd(L, m, k), rnd(L, k, r), rnd(L, m, r)
Z = torch.empty((L, m, r), dtype=torch.int64, device="cuda")
D, E = rnd(m, k), rnd(k, r)
for _ in range(2):
    K.beaver_gemm_sim(Z, m * r, 0, C.data_ptr(), m * r, 0, X.data_ptr(), X.stride(0), X.stride(1), X.stride(2), 0,
                      A.data_ptr(), m * k, 0, Y.data_ptr(), Y.stride(0), Y.stride(1), Y.stride(2), 0, B.data_ptr(),
                      k * r, 0, L, 1, m, k, r, 0, 64)
    K.beaver_gemm(Z, m * r, C.data_ptr(), m * r, D, E, A.data_ptr(), m * k, B.data_ptr(), k * r, L, m, k, r, 0, 64)
torch.cuda.synchronize()
