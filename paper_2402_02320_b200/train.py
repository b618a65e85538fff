"""Secure CNN / MLP training on secret shares (BASELINE configs 0-2).

The reference package has no training or convolution code; the
paper trains Simple / LeNet / AlexNet / VGG16m with Piranha's recipe
(layer tables :1289-1458). Everything here is a
composition of the reference's pinned primitives, so parity is pinned per
primitive (and the composition is restated in ``oracle/train_sim.py`` for a
bit-exact end-to-end check):

* weights and activations are additive shares at precision p (w = 64);
* Conv2d = im2col (local kernel) + Beaver matmul with the secret weight
  matrix (one matrix triple, ``basic.py:45-79``) + secret bias + truncation;
* AvgPool2d (power-of-two window) = local window sum + truncation;
* ReLU = gt / bit2a / mul (``nn.py:92-97``), keeping the converted sign bit
  so the backward pass is one Beaver mul;
* Linear = Beaver matmul with secret weights + secret bias + truncation;
* softmax-cross-entropy gradient = softmax (``nn.py:139-147``) - one-hot;
* SGD with lr = 2^-lr_shift and batch 2^b folds 1/B into one truncation of
  the doubled-precision gradient: W -= trunc(dW_2p, p + lr_shift + b).

Both backward matmuls of a layer (dW = X^T dZ, dX = dZ W^T) open in ONE round.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .nn import softmax
from .protocols import batch_matmul, bit2a, gt, mul, scale_fixed, truncate
from .sharing import AShare, public_ashare


def _transpose(x: AShare) -> AShare:
    """Transposed VIEW (no copy): batch_matmul masks it with mpx_mask_sub_t."""
    return AShare.strided(x.values.transpose(-1, -2), x.width, x.frac, x.parties)


def _colsum(session, z: AShare) -> AShare:
    """sum over rows of a (rows, C) share -> (C,) (local ring sum)."""
    r, c = z.shape
    out = session.alloc((session.L, c))
    K.ring_colsum(out, z.values.contiguous(), session.L, r, c, z.width)
    return AShare(out, z.width, z.frac, session.parties)


def _fused_layer(s) -> bool:
    """Sim mode with the layer-plumbing kernels (all parties local, L <= 8)."""
    return s.fused and getattr(s, "fuse_ops", True) and s.L <= 8


def _trunc_takes(s, n: int, f: int, w: int):
    """Material + ledger of one signed truncation, in _truncate_core's order
    (derived.py:20-70): edaBit(w, f) arithmetic, edaBit(w, w-1-f), one round."""
    from .session import arith_payload
    r_lo, _ = s.store.take_edabits(w, f, n, need_bits=False)
    hw = w - 1 - f
    r_hi = s.store.take_edabits(w, hw, n, need_bits=False)[0] if hw > 0 else None
    s.exchange(payload=arith_payload(w, n))
    s.metrics.count(trunc_count=1)
    return (r_lo.ptr, r_lo.ps), ((r_hi.ptr, r_hi.ps) if r_hi is not None else (None, 0))


def _trunc_bias_out(s, z: AShare, b: AShare, p: int, B: int, S: int, nchw: bool, out_shape) -> AShare:
    """trunc(z + lift(b), p) in one kernel; nchw stores the conv output layout."""
    w = z.width
    out = s.alloc((s.L,) + tuple(out_shape))
    (lo, lo_ps), (hi, hi_ps) = _trunc_takes(s, z.size, p, w)
    K.trunc_rows_bias(out, z.values, b.values.contiguous() if b is not None else None, p, lo, lo_ps, hi, hi_ps, s.L,
                      B, S, z.shape[-1], nchw, w, p, 1 << (w - 2), 1 << (w - 2 - p), s.p0)
    return AShare(out, w, z.frac - p, s.parties)


def _add_bias(session, z: AShare, b: AShare, p: int) -> AShare:
    """z + broadcast(b * 2^p) over rows, in place on the fresh product z."""
    rows, cols = z.shape
    K.ring_add_rowvec(z.values, b.values.contiguous(), session.L, rows, cols, p, z.width)
    return z


@dataclass
class InitSpec:
    seed: int = 7
    frac: int = 23
    width: int = 64


def _kaiming(rng, fan_in, shape):
    return rng.normal(0.0, math.sqrt(2.0 / fan_in), size=shape)


class Layer:
    params: tuple = ()

    def step(self, session, shift: int) -> None:
        pass


class Conv2d(Layer):
    """(C_in -> C_out, K x K, stride, pad); weight matrix (C_in*K*K, C_out)."""

    def __init__(self, session, cin, cout, k, stride=1, pad=0, *, rng, name, spec: InitSpec, bias: bool = True):
        self.cin, self.cout, self.k, self.stride, self.pad = cin, cout, k, stride, pad
        self.p = spec.frac
        fan_in = cin * k * k
        self.W = session.share_fixed(_kaiming(rng, fan_in, (fan_in, cout)), spec.width, spec.frac,
                                     _key(spec, name + ".W"))
        if bias:
            self.b = session.share_fixed(np.zeros(cout), spec.width, spec.frac, _key(spec, name + ".b"))

    def forward(self, s, x: AShare) -> AShare:
        B, C, H, W = x.shape
        k, st, pd = self.k, self.stride, self.pad
        OH, OW = (H + 2 * pd - k) // st + 1, (W + 2 * pd - k) // st + 1
        rows, cols = B * OH * OW, C * k * k
        cv = s.alloc((s.L, rows, cols))
        K.im2col(cv, x.values, s.L, B, C, H, W, k, st, pd)
        self.cols = AShare(cv, x.width, x.frac, s.parties)
        self.in_shape = (B, C, H, W)
        z = batch_matmul(s, [(self.cols, self.W)])[0]
        self.out_hw = (OH, OW)
        b = getattr(self, "b", None)
        if _fused_layer(s) and s.L <= 4:   # the NCHW epilogue's smem tiles hold <= 4 parties
            return _trunc_bias_out(s, z, b, self.p, B, OH * OW, True, (B, self.cout, OH, OW))
        z = truncate(s, _add_bias(s, z, b, self.p) if b is not None else z, self.p)
        v = z.values.view(s.L, B, OH, OW, self.cout).permute(0, 1, 4, 2, 3).contiguous()
        return AShare(v, z.width, z.frac, s.parties)

    def backward(self, s, dy: AShare, need_dx: bool = True) -> AShare | None:
        B, C, H, W = self.in_shape
        OH, OW = self.out_hw
        dz = AShare(dy.values.permute(0, 1, 3, 4, 2).reshape(s.L, B * OH * OW, self.cout).contiguous(),
                    dy.width, dy.frac, s.parties)
        pairs = [(_transpose(self.cols), dz)]
        if need_dx:
            pairs.append((dz, _transpose(self.W)))
        outs = batch_matmul(s, pairs)
        self.gW = outs[0]
        if hasattr(self, "b"):
            self.gb = _colsum(s, dz)
        if not need_dx:
            return None
        dcols = truncate(s, outs[1], self.p)
        dx = s.alloc((s.L, B, C, H, W))
        K.col2im(dx, dcols.values, s.L, B, C, H, W, self.k, self.stride, self.pad, dcols.width)
        return AShare(dx, dcols.width, dcols.frac, s.parties)

    def step(self, s, shift: int) -> None:
        self.W = self.W - truncate(s, self.gW, self.p + shift, out_frac=self.p)
        if hasattr(self, "b"):
            self.b = self.b - truncate(s, self.gb, shift, out_frac=self.p)


class AvgPool2d(Layer):
    """k x k average pool, stride st (default k; PAPER.md:1348-1458 uses 3x3/2
    and 2x2/1 too): window sum, then / k^2 as a truncation by log2(k^2) for
    power-of-two windows, else a public fixed-point 1/k^2 scale + truncation
    by p. Backward: the same scaling of dy, scattered over the windows."""

    def __init__(self, k: int = 2, stride: int | None = None):
        self.k = k
        self.st = k if stride is None else stride
        area = k * k
        self.shift = area.bit_length() - 1 if area & (area - 1) == 0 else None

    def _scale(self, s, v: AShare) -> AShare:
        if self.shift is not None:
            return truncate(s, v, self.shift, out_frac=v.frac)
        return truncate(s, scale_fixed(s, v, 1.0 / (self.k * self.k)), v.frac)

    def _out_hw(self, H, W):
        return (H - self.k) // self.st + 1, (W - self.k) // self.st + 1

    def forward(self, s, x: AShare) -> AShare:
        B, C, H, W = x.shape
        OH, OW = self._out_hw(H, W)
        out = s.alloc((s.L, B, C, OH, OW))
        K.ring_pool_sum(out, x.values.contiguous(), s.L * B * C, H, W, self.k, x.width, stride=self.st)
        self.in_shape = (B, C, H, W)
        return self._scale(s, AShare(out, x.width, x.frac, s.parties))

    rows_out = False   # set by Model when a Conv2d precedes: emit the conv's row layout

    def backward(self, s, dy: AShare, need_dx: bool = True) -> AShare:
        B, C, H, W = self.in_shape
        k = self.k
        if self.rows_out and _fused_layer(s) and self.shift is not None and self.st == k \
                and H % k == 0 and W % k == 0:
            z = s.alloc((s.L, B * H * W, C))
            (lo, lo_ps), (hi, hi_ps) = _trunc_takes(s, dy.size, self.shift, dy.width)
            w = dy.width
            K.trunc_expand_rows(z, dy.values.contiguous(), lo, lo_ps, hi, hi_ps, s.L, B, C, H // k, W // k, k, w,
                                self.shift, 1 << (w - 2), 1 << (w - 2 - self.shift), s.p0)
            # logical NCHW view of the row-layout buffer: the conv backward's
            # permute back to rows is then free
            return AShare.strided(z.view(s.L, B, H, W, C).permute(0, 1, 4, 2, 3), w, dy.frac, s.parties)
        d = self._scale(s, dy)
        dx = s.alloc((s.L, B, C, H, W))
        K.ring_pool_scatter(dx, d.values.contiguous(), s.L * B * C, H, W, k, self.st, d.width)
        return AShare(dx, d.width, d.frac, s.parties)


class ReLU(Layer):
    def forward(self, s, x: AShare) -> AShare:
        from . import fused as F
        if F.fusable_cmp(s, x):
            y, self.sign = F.relu_fused(s, x, ReLU._protocol, want_sign=True)
            return y
        return self._protocol(s, x, self)

    @staticmethod
    def _protocol(s, x: AShare, layer=None) -> AShare:
        zero = public_ashare(0, x.width, x.frac, s, shape=x.shape)
        sign = bit2a(s, gt(s, x, zero), x.width)
        if layer is not None:
            layer.sign = sign
        return mul(s, sign, x)

    def backward(self, s, dy: AShare, need_dx: bool = True) -> AShare:
        return mul(s, self.sign, dy)


class Flatten(Layer):
    def forward(self, s, x: AShare) -> AShare:
        self.in_shape = x.shape
        return x.reshape((x.shape[0], math.prod(x.shape[1:])))

    def backward(self, s, dy: AShare, need_dx: bool = True) -> AShare:
        return dy.reshape(self.in_shape)


class Linear(Layer):
    def __init__(self, session, fin, fout, *, rng, name, spec: InitSpec, bias: bool = True):
        self.p = spec.frac
        self.W = session.share_fixed(_kaiming(rng, fin, (fin, fout)), spec.width, spec.frac,
                                     _key(spec, name + ".W"))
        if bias:
            self.b = session.share_fixed(np.zeros(fout), spec.width, spec.frac, _key(spec, name + ".b"))

    def forward(self, s, x: AShare) -> AShare:
        self.x = x
        z = batch_matmul(s, [(x, self.W)])[0]
        b = getattr(self, "b", None)
        if _fused_layer(s):
            return _trunc_bias_out(s, z, b, self.p, z.shape[0], 1, False, z.shape)
        return truncate(s, _add_bias(s, z, b, self.p) if b is not None else z, self.p)

    def backward(self, s, dy: AShare, need_dx: bool = True) -> AShare | None:
        pairs = [(_transpose(self.x), dy)]
        if need_dx:
            pairs.append((dy, _transpose(self.W)))
        outs = batch_matmul(s, pairs)
        self.gW = outs[0]
        if hasattr(self, "b"):
            self.gb = _colsum(s, dy)
        return truncate(s, outs[1], self.p) if need_dx else None

    def step(self, s, shift: int) -> None:
        self.W = self.W - truncate(s, self.gW, self.p + shift, out_frac=self.p)
        if hasattr(self, "b"):
            self.b = self.b - truncate(s, self.gb, shift, out_frac=self.p)


def _key(spec: InitSpec, label: str):
    import hashlib
    tag = hashlib.sha256(f"{spec.seed}:param:{label}".encode()).digest()
    return [int.from_bytes(tag[:8], "little"), int.from_bytes(tag[8:16], "little")]


class Model:
    """Sequential secure model with a softmax-cross-entropy head."""

    @property
    def n_params(self) -> int:
        return sum(getattr(layer, nm).size for layer in self.layers for nm in ("W", "b") if hasattr(layer, nm))

    def __init__(self, layers):
        self.layers = list(layers)
        for prev, layer in zip(self.layers, self.layers[1:]):
            if isinstance(layer, AvgPool2d) and isinstance(prev, Conv2d):
                layer.rows_out = True

    def forward(self, s, x: AShare) -> AShare:
        for layer in self.layers:
            x = layer.forward(s, x)
        return x

    def train_step(self, s, x: AShare, y_onehot: AShare, lr_shift: int) -> AShare:
        """One SGD step on a batch (batch size must be a power of two).
        Returns the logits (shares) of the forward pass."""
        B = x.shape[0]
        bshift = int(round(math.log2(B)))
        if (1 << bshift) != B:
            raise ValueError("batch size must be a power of two")
        with s.scope("forward"):
            logits = self.forward(s, x)
        with s.scope("loss"):
            dz = softmax(s, logits) - y_onehot
        with s.scope("backward"):
            g = dz
            for i in range(len(self.layers) - 1, -1, -1):
                g = self.layers[i].backward(s, g, need_dx=i > 0)
        with s.scope("sgd"):
            _sgd(s, self.layers, lr_shift + bshift)
        return logits


def _sgd(s, layers, shift: int) -> None:
    """W -= trunc(dW_2p, p + shift), b -= trunc(db, shift) for every layer.
    Sim mode: all truncations in ONE launch (mpx_trunc_sub_multi), same
    material order, rounds and ledger as the per-layer path (derived.py:20-70)."""
    jobs = [(layer, nm, getattr(layer, g), f) for layer in layers if hasattr(layer, "W")
            for nm, g, f in (("W", "gW", layer.p + shift), ("b", "gb", shift)) if hasattr(layer, nm)]
    if not (s.fused and getattr(s, "fuse_ops", True) and jobs and len(jobs) <= K.TRUNC_JOBS_MAX and s.L <= 16
            and all(g.width == 64 for _, _, g, _ in jobs)):
        for layer in layers:
            layer.step(s, shift)
        return
    from .session import arith_payload
    w = 64
    kj = []
    for layer, nm, g, f in jobs:
        n = g.size
        r_lo, _ = s.store.take_edabits(w, f, n, need_bits=False)
        hw = w - 1 - f
        r_hi = s.store.take_edabits(w, hw, n, need_bits=False)[0] if hw > 0 else None
        base = getattr(layer, nm)
        # in place: each element is read and written by the same thread
        z = base.values if base.values.is_contiguous() else s.alloc((s.L,) + g.shape)
        kj.append({"z": z, "base": base.values.contiguous(), "x": g.values.contiguous(), "r_lo": r_lo.ptr,
                   "lo_ps": r_lo.ps, "r_hi": r_hi.ptr if r_hi is not None else None,
                   "hi_ps": r_hi.ps if r_hi is not None else 0, "n": n, "f": f,
                   "bias": 1 << (w - 2), "unbias": 1 << (w - 2 - f)})
        s.exchange(payload=arith_payload(w, n))
        s.metrics.count(trunc_count=1)
        if z is not base.values:
            setattr(layer, nm, AShare(z, w, base.frac, s.parties))
    K.trunc_sub_multi(kj, s.L, w, s.p0)


def lenet(session, spec: InitSpec = InitSpec()) -> Model:
    """Paper Table 'LeNet': conv(20,5x5) pool ReLU conv(50,5x5) pool ReLU FC800x500 ReLU
    FC500x10 — 430,500 weights, no biases (the table's count)."""
    rng = np.random.default_rng(spec.seed)
    kw = dict(rng=rng, spec=spec, bias=False)
    return Model([Conv2d(session, 1, 20, 5, name="conv1", **kw), AvgPool2d(2), ReLU(),
                  Conv2d(session, 20, 50, 5, name="conv2", **kw), AvgPool2d(2), ReLU(), Flatten(),
                  Linear(session, 800, 500, name="fc1", **kw), ReLU(),
                  Linear(session, 500, 10, name="fc2", **kw)])


def alexnet(session, spec: InitSpec = InitSpec()) -> Model:
    """Paper Table 'AlexNet' on CIFAR-10 3x32x32: 2,552,874
    parameters = bias-free convolutions + fully-connected layers with bias."""
    rng = np.random.default_rng(spec.seed)
    kw = dict(rng=rng, spec=spec)
    return Model([Conv2d(session, 3, 96, 11, 4, 9, name="conv1", bias=False, **kw), AvgPool2d(3, 2), ReLU(),
                  Conv2d(session, 96, 256, 5, 1, 1, name="conv2", bias=False, **kw), AvgPool2d(2, 1), ReLU(),
                  Conv2d(session, 256, 384, 3, 1, 1, name="conv3", bias=False, **kw), ReLU(),
                  Conv2d(session, 384, 256, 3, 1, 1, name="conv4", bias=False, **kw), ReLU(), Flatten(),
                  Linear(session, 256, 256, name="fc1", **kw), ReLU(),
                  Linear(session, 256, 256, name="fc2", **kw), ReLU(),
                  Linear(session, 256, 10, name="fc3", **kw)])


def vgg16m(session, spec: InitSpec = InitSpec(frac=26)) -> Model:
    """Paper Table 'VGG16m' on CIFAR-10 3x32x32, p = 26:
    nine bias-free 3x3 convolutions with five 2x2 average pools, three
    fully-connected layers with bias — 7,242,442 parameters as the table's
    layer list gives them (its caption says 7,439,306; the listed layers do
    not reach that count with or without biases)."""
    rng = np.random.default_rng(spec.seed)
    kw = dict(rng=rng, spec=spec)
    layers, cin = [], 3
    for i, (cout, pool) in enumerate([(64, False), (64, True), (128, False), (128, True), (256, False),
                                      (256, True), (512, False), (512, True), (512, True)]):
        layers.append(Conv2d(session, cin, cout, 3, 1, 1, name=f"conv{i + 1}", bias=False, **kw))
        if pool:
            layers.append(AvgPool2d(2))
        layers.append(ReLU())
        cin = cout
    layers += [Flatten(), Linear(session, 512, 256, name="fc1", **kw), ReLU(),
               Linear(session, 256, 256, name="fc2", **kw), ReLU(),
               Linear(session, 256, 10, name="fc3", **kw)]
    return Model(layers)


def simple_mlp(session, spec: InitSpec = InitSpec()) -> Model:
    """Paper Table 'Simple network': 784-128-128-10 with ReLU."""
    rng = np.random.default_rng(spec.seed)
    return Model([Linear(session, 784, 128, rng=rng, name="fc1", spec=spec), ReLU(),
                  Linear(session, 128, 128, rng=rng, name="fc2", spec=spec), ReLU(),
                  Linear(session, 128, 10, rng=rng, name="fc3", spec=spec)])


class GraphedStep:
    """One secure training step captured in a CUDA graph and replayed.

    The ~150 rounds / ~330 kernel launches of a LeNet step are issued once at
    capture; a replay costs one graph launch. Every pointer the step touches is
    stable: inputs and weights live in static buffers (updated weights are
    copied back inside the graph), intermediates come from the graph's private
    pool, and the dealer re-deals fresh material into the SAME store arrays
    before each replay (``DealerGraph.redeal``: the whole re-deal is its own
    CUDA graph, keys in device slots), outside the step's graph.

    Construction runs one eager warm-up step (seed0 material) and then
    restores the weights it updated, so the model is where the caller left
    it: the first ``step()`` is the model's first update.
    """

    def __init__(self, session, model: Model, x: AShare, y: AShare, lr_shift: int, demands: dict,
                 needs_bits: dict, seed0: int, capture_error_mode: str = "global"):
        from .preprocessing import DealerGraph, device_store
        self.s, self.model, self.lr_shift = session, model, lr_shift
        self.demands, self.needs_bits = demands, needs_bits
        self.params = [(layer, nm) for layer in model.layers for nm in ("W", "b") if hasattr(layer, nm)]
        self.bufs = [getattr(layer, nm) for layer, nm in self.params]
        self.x, self.y = x, y
        session.store = device_store(seed0, session.n_parties, demands, parties=session.parties,
                                     device=session.device, needs_bits=needs_bits)
        self.dealer = DealerGraph(session.store, demands, needs_bits, seed0)
        # warm-up (eager) step: first-use work (attributes, schedules) happens
        # here; the weights it updates are restored afterwards
        snapshot = [b.values.clone() for b in self.bufs]
        side = torch.cuda.Stream(session.device)
        side.wait_stream(torch.cuda.current_stream(session.device))
        with torch.cuda.stream(side):
            model.train_step(session, x, y, lr_shift)
            self._writeback()
        torch.cuda.current_stream(session.device).wait_stream(side)
        torch.cuda.synchronize(session.device)
        for b, v in zip(self.bufs, snapshot):
            b.values.copy_(v)
        del snapshot
        session.store.rewind()
        self.graph = torch.cuda.CUDAGraph()
        # party sessions: the round's NCCL collectives are captured as graph
        # nodes too ("thread_local": other threads, e.g. NCCL's watchdog, may
        # keep querying their own events during the capture)
        with torch.cuda.graph(self.graph, capture_error_mode=capture_error_mode):
            self.logits = model.train_step(session, x, y, lr_shift)
            self._writeback()

    def _writeback(self):
        for (layer, nm), buf in zip(self.params, self.bufs):
            cur = getattr(layer, nm)
            if cur is not buf:
                buf.values.copy_(cur.values)
                setattr(layer, nm, buf)

    def step(self, seed: int) -> AShare:
        """Re-deal fresh material in place (the dealer's own CUDA graph), replay the captured step."""
        self.dealer.redeal(seed)
        self.graph.replay()
        return self.logits
