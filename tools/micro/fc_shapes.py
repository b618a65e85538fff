"""Time the fused SIMT Beaver kernel (mpx_beaver_gemm_sim) on LeNet's FC-layer
product shapes (fc2 forward / dW / dX at three parties), each captured in a
CUDA graph so launch overhead is excluded.
    python tools/micro/fc_shapes.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import kernels as Kn  # noqa: E402

L = 3
g = torch.Generator(device="cuda").manual_seed(1)
rnd = lambda *s: torch.randint(-2**62, 2**62, s, device="cuda", generator=g)  # noqa: E731
for name, (M, K, N) in {"fc2 fwd": (128, 500, 10), "fc2 dW": (500, 128, 10), "fc2 dX": (128, 10, 500),
                        "fc1 fwd": (128, 800, 500)}.items():
    X, A, C, Y, B = rnd(L, M, K), rnd(L, M, K), rnd(L, M, N), rnd(L, K, N), rnd(L, K, N)
    Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
    fn = lambda: Kn.beaver_gemm_sim(Z, M * N, L * M * N, C.data_ptr(), M * N, 0, X.data_ptr(), M * K, K, 1, 0,  # noqa
                                    A.data_ptr(), M * K, 0, Y.data_ptr(), K * N, N, 1, 0, B.data_ptr(), K * N, 0,
                                    L, 1, M, K, N, 0, 64)
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(10):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} {M}x{K}x{N}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per product (graph)")

if os.environ.get("FC_SWEEP"):
    # every tile config (MPX_BS_CFG) on the same shapes
    for cfg in range(7):
        os.environ["MPX_BS_CFG"] = str(cfg)
        for name, (M, K, N) in {"fc2 fwd": (128, 500, 10), "fc2 dW": (500, 128, 10), "fc2 dX": (128, 10, 500)}.items():
            X, A, C, Y, B = rnd(L, M, K), rnd(L, M, K), rnd(L, M, N), rnd(L, K, N), rnd(L, K, N)
            Z = torch.empty((L, M, N), dtype=torch.int64, device="cuda")
            fn = lambda: Kn.beaver_gemm_sim(Z, M * N, L * M * N, C.data_ptr(), M * N, 0, X.data_ptr(), M * K, K, 1,  # noqa
                                            0, A.data_ptr(), M * K, 0, Y.data_ptr(), K * N, N, 1, 0, B.data_ptr(),
                                            K * N, 0, L, 1, M, K, N, 0, 64)
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                fn()
            e1.record()
            torch.cuda.synchronize()
            print(f"cfg {cfg} {name}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us (eager)")
    os.environ.pop("MPX_BS_CFG")
