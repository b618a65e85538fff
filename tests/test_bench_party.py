"""GPU (1 device): bench.py's N>1 path — one PartySession per party, per-round
kernels, exchanges, max-over-ranks timing, e2e streaming — run with 2 party
threads on one GPU through a ThreadHub instead of NCCL (no device-side
waiting). Checks the JSON line and that the opened result is correct."""

import io
import json
import threading
import contextlib
import types

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


class ThreadGroup:
    def __init__(self, hub, rank, world):
        self.hub, self.rank, self.world, self.local = hub, rank, world, 0
        self._vals = hub.vals

    def init(self, dev):
        pass

    def comm(self):
        return self.hub.comm(self.rank)

    def barrier(self):
        torch.cuda.synchronize()
        self.hub.barrier.wait()

    def max(self, v, dev):
        self._vals[self.rank] = v
        self.hub.barrier.wait()
        m = max(self._vals)
        self.hub.barrier.wait()
        return m

    def close(self):
        pass


def test_bench_party_path_two_threads():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    from paper_2402_02320_b200.session import ThreadHub
    hub = ThreadHub(2)
    hub.barrier = threading.Barrier(2, timeout=300)
    hub.vals = [0.0, 0.0]
    args = types.SimpleNamespace(gpus=2, steps=2, warmup=1, batch=8, cpu_sample=0, no_cpu=True,
                                 no_sweep=True, chunks=4, impl="b200")
    outs, errs = {}, {}

    def worker(r):
        try:
            outs[r] = bench.run_b200(args, ThreadGroup(hub, r, 2))
        except BaseException as e:  # noqa: BLE001
            errs[r] = e
            hub.barrier.abort()

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[min(errs)]
    line = outs[0]
    assert outs[1] is None
    json.dumps(line)
    assert line["n_gpus"] == 2 and line["config"]["parties"] == 2
    assert all(np.isfinite(line["loss_first_last"]))
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches_per_step"] > 100
