"""conv1 weight-gradient product (25 x 73728 x 20, 3 parties, X = im2col^T view)
on the tiled SIMT sim kernel (mpx_beaver_gemm_sim); MPX_LIB selects A/B builds."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import kernels as Kn  # noqa: E402
L, M, K, N = 3, 25, 73728, 20
g = torch.Generator(device="cuda").manual_seed(1)
rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
XT, A, C, Y, B = rnd(L, K, M), rnd(L, M, K), rnd(L, M, N), rnd(L, K, N), rnd(L, K, N)
Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
f = lambda: Kn.beaver_gemm_sim(Z, M * N, L * M * N, C.data_ptr(), M * N, 0, XT.data_ptr(), K * M, 1, M, 0,  # noqa
                               A.data_ptr(), M * K, 0, Y.data_ptr(), K * N, N, 1, 0, B.data_ptr(), K * N, 0, L, 1, M,
                               K, N, 0, 64)
for _ in range(3):
    f()
torch.cuda.synchronize()
ref = Z.clone()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20):
    f()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"{os.path.basename(os.environ.get('MPX_LIB', 'libmpx.so'))}: {us:.1f} us  checksum {int(ref.sum())}")
