"""CPU, world_size 2 over gloo: the party layer's collectives (int64 sum with
Z_2^64 wrap, rank-ordered all-gather) and each rank's party-mode dry run
(material demand + ledger == the reference's) across real processes."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_02320_b200.preprocessing import DemandCounter
        from paper_2402_02320_b200.session import DistComm, PartySession, demands_by_name
        from cases import CASES
        from gpu_engine import GpuEngine
        comm = DistComm()
        # 1) int64 sum wraps mod 2^64 exactly like the ring
        big = np.array([(1 << 63) - 5, 12345, -7, 1 << 62], dtype=np.int64)
        t = torch.from_numpy(big * (rank + 1))
        comm.allreduce_sum_(t)
        want = (big.astype(object) * 3) % (1 << 64)
        ok_sum = [int(v) % (1 << 64) for v in t.tolist()] == [int(v) for v in want]
        # 2) all-gather is rank ordered
        g = comm.allgather(torch.full((5,), rank * 10 + 1, dtype=torch.int64))
        ok_gather = g.tolist() == [[1] * 5, [11] * 5]
        # 3) party-mode dry run per rank == reference demand + ledger
        eng = GpuEngine()
        res = {}
        for name in ("reciprocal", "softmax", "batch_matmul", "relu"):
            fn, n = CASES[name]
            if n != world:
                fn, n = CASES[name][0], world
            counter = DemandCounter((rank,), world)
            s = PartySession(rank, world, comm, counter)
            fn(eng, s)
            res[name] = (demands_by_name(counter), s.metrics.total.as_dict(),
                         {k: v.as_dict() for k, v in sorted(s.metrics.ledger.items())},
                         dict(s.metrics.bytes_per_peer))
        q.put((rank, ok_sum, ok_gather, res))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_party_layer():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, ok_sum, ok_gather, res in got:
        assert ok_sum and ok_gather, rank
        for name, (dem, total, ledger, per_peer) in res.items():
            z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
            info = json.loads(bytes(z["info"]).decode())
            if int(z["n"]) == 2:
                assert dem == info["demands"], name
                assert total == info["total"], name
                assert ledger == info["ledger"], name
            assert list(per_peer) == [1 - rank]
            assert per_peer[1 - rank] == total["bytes"]
