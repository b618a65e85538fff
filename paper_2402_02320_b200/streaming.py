"""Host-buffer entry point: stream an elementwise secure op over chunks.

``run_host(op, session, x_host, width, frac)`` is the public API call for
inputs that live in (pinned) host memory: the element range is split into
chunks and three CUDA streams overlap the host->device copy of chunk k+1, the
secure op on chunk k and the device->host copy of chunk k-1. Each chunk is one
ordinary protocol call (same rounds, ledger and material kinds per element as
one call over the whole batch; the material is consumed chunk by chunk).
"""

from __future__ import annotations

import torch

from .sharing import AShare

_STREAMS: dict = {}


def _streams(dev):
    """Three long-lived side streams per device (the caching allocator keeps
    per-stream pools, so fresh streams per call would force cudaMalloc)."""
    key = torch.device(dev).index
    if key not in _STREAMS:
        _STREAMS[key] = tuple(torch.cuda.Stream(dev) for _ in range(3))
    return _STREAMS[key]


def run_host(op, session, x_host: torch.Tensor, width: int, frac: int, chunks: int = 8,
             y_host: torch.Tensor | None = None) -> torch.Tensor:
    """x_host: int64[L, N] pinned shares of the local parties -> int64[L, N] pinned."""
    L, N = x_host.shape
    dev = session.device
    if y_host is None:
        y_host = torch.empty_like(x_host).pin_memory()
    chunks = max(1, min(chunks, N))
    bounds = [N * k // chunks for k in range(chunks + 1)]
    h2d, comp, d2h = _streams(dev)
    main = torch.cuda.current_stream(dev)
    h2d.wait_stream(main)
    comp.wait_stream(main)
    xs, ys, ev_in, ev_out = [], [], [], []
    for k in range(chunks):
        c0, c1 = bounds[k], bounds[k + 1]
        xd = torch.empty((L, c1 - c0), dtype=torch.int64, device=dev)
        with torch.cuda.stream(h2d):
            for l in range(L):
                xd[l].copy_(x_host[l, c0:c1], non_blocking=True)
            e = torch.cuda.Event()
            e.record(h2d)
        xs.append(xd)
        ev_in.append(e)
    for k in range(chunks):
        with torch.cuda.stream(comp):
            comp.wait_event(ev_in[k])
            y = op(session, AShare(xs[k], width, frac, session.parties))
            e = torch.cuda.Event()
            e.record(comp)
        ys.append(y)
        ev_out.append(e)
        c0, c1 = bounds[k], bounds[k + 1]
        with torch.cuda.stream(d2h):
            d2h.wait_event(e)
            for l in range(L):
                y_host[l, c0:c1].copy_(y.values[l], non_blocking=True)
    main.wait_stream(d2h)
    for t in xs + [y.values for y in ys]:
        t.record_stream(d2h)
    return y_host
