"""Party layer (one party per GPU): a round's payloads share one
buffer and are opened by ONE collective in place (no concatenation), on gloo
world 2 (CPU) - and on the GPU, the one-party (L = 1) LeNet step with the
collectives elided (LoopbackComm) runs inside a CUDA graph with exactly the
sim run's rounds."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_02320_b200.session import _covering


def test_covering_views():
    buf = torch.arange(12, dtype=torch.int64)
    a, b, c = buf[0:4], buf[4:7], buf[7:12]
    cov = _covering([c, a, b])                      # any order
    assert cov is not None and cov.numel() == 12 and cov.data_ptr() == buf.data_ptr()
    assert _covering([a, c]) is None                # gap
    assert _covering([buf.view(3, 4)[:, 1]]) is None   # strided
    assert _covering([buf.view(2, 6).unbind(0)[1]]).numel() == 6
    other = torch.arange(3, dtype=torch.int64)
    assert _covering([a, other]) is None            # two storages


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_02320_b200.preprocessing import DemandCounter
        from paper_2402_02320_b200.session import DistComm, PartySession
        s = PartySession(rank, world, DistComm(), DemandCounter((rank,), world), device=torch.device("cpu"))
        s.dry = False                                  # exercise the collective on real CPU tensors
        pay = torch.full((2, 5), rank + 1, dtype=torch.int64)
        pay[1] *= 10
        d, e = pay.unbind(0)
        od, oe = s._collective([d, e], [])
        contiguous = od.data_ptr() == d.data_ptr() and od.tolist() == [3] * 5 and oe.tolist() == [30] * 5
        x, y = torch.full((3,), rank + 1, dtype=torch.int64), torch.full((4,), 7 * (rank + 1), dtype=torch.int64)
        ox, oy = s._collective([x, y], [])              # separate buffers: concatenated path
        separate = ox.tolist() == [3] * 3 and oy.tolist() == [21] * 4
        q.put((rank, contiguous, separate, s.metrics.physical_bytes))
    finally:
        dist.destroy_process_group()


def test_round_payload_single_collective_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, contiguous, separate, phys in res:
        assert contiguous and separate, rank
        assert phys == 8 * (10 + 7)


@pytest.mark.gpu
def test_loopback_party_step_graph():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    from paper_2402_02320_b200 import train
    from paper_2402_02320_b200.preprocessing import DemandCounter
    from paper_2402_02320_b200.session import SimSession
    out = bench.party_mode_entry(torch, torch.device("cuda", 0), n=2, steps=2, warmup=1)
    x, y = bench.lenet_data(bench.BATCH)
    c = DemandCounter((0, 1), 2)
    sd = SimSession(2, c)
    train.lenet(sd).train_step(sd, sd.share_fixed(x, 64, 23, [1, 1]), sd.share_fixed(y, 64, 23, [1, 2]), 5)
    assert out["rounds_per_step"] == sd.metrics.total.rounds
    assert out["local_compute_ms_per_step"] > 0 and out["collective_bytes_per_step"] > 0
