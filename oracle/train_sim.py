"""CPU oracle for secure training — TEST INFRASTRUCTURE ONLY.

Restates ``paper_2402_02320_b200/train.py`` (Conv2d / AvgPool2d / ReLU /
Linear / softmax-CE / SGD) over the oracle's primitives, which are pinned
bit-exactly to the reference (``tests/test_oracle_golden.py``). The reference
itself has no training or convolution code, so training parity
is pinned per primitive; this restatement lets the tests check a whole GPU
training step bit-for-bit on every party's shares.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

from . import mpc_sim as O

U64 = np.uint64


def im2col(x: np.ndarray, k: int, stride: int, pad: int) -> np.ndarray:
    """x: (n, B, C, H, W) -> (n, B*OH*OW, C*k*k), zero padded."""
    n, B, C, H, W = x.shape
    OH, OW = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    xp = np.zeros((n, B, C, H + 2 * pad, W + 2 * pad), U64)
    xp[:, :, :, pad:pad + H, pad:pad + W] = x
    out = np.empty((n, B, OH, OW, C, k, k), U64)
    for kh in range(k):
        for kw in range(k):
            out[:, :, :, :, :, kh, kw] = xp[:, :, :, kh:kh + stride * OH:stride,
                                            kw:kw + stride * OW:stride].transpose(0, 1, 3, 4, 2)
    return out.reshape(n, B * OH * OW, C * k * k)


def col2im(cols: np.ndarray, shape, k: int, stride: int, pad: int, width: int) -> np.ndarray:
    """Adjoint of im2col: scatter-add (mod 2^w) into (n, B, C, H, W)."""
    n, B, C, H, W = shape
    OH, OW = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    c = cols.reshape(n, B, OH, OW, C, k, k)
    xp = np.zeros((n, B, C, H + 2 * pad, W + 2 * pad), U64)
    with np.errstate(over="ignore"):
        for kh in range(k):
            for kw in range(k):
                xp[:, :, :, kh:kh + stride * OH:stride, kw:kw + stride * OW:stride] += \
                    c[:, :, :, :, :, kh, kw].transpose(0, 1, 4, 2, 3)
    return O.wrap(xp[:, :, :, pad:pad + H, pad:pad + W].copy(), width)


def _key(seed, label):
    tag = hashlib.sha256(f"{seed}:param:{label}".encode()).digest()
    return [int.from_bytes(tag[:8], "little"), int.from_bytes(tag[8:16], "little")]


def share_fixed(s: O.Sim, floats, width, frac, key) -> O.AShare:
    enc = O.encode(np.asarray(floats, np.float64), width, frac)
    return O.AShare(O.deal_inputs_arith(enc, s.n, width, key), width, frac)


def _T(x: O.AShare) -> O.AShare:
    return O.AShare(np.ascontiguousarray(x.values.swapaxes(-1, -2)), x.width, x.frac)


def _bcast_rows(b: O.AShare, rows) -> O.AShare:
    return O.AShare(np.ascontiguousarray(np.broadcast_to(b.values[:, None, :], (b.values.shape[0], rows,
                                                                               b.values.shape[1]))),
                    b.width, b.frac)


def _lift(x: O.AShare, p) -> O.AShare:
    return x.mul_public(1 << p, frac_delta=p)


def _colsum(z: O.AShare) -> O.AShare:
    return O.AShare(O.rsum(z.values, z.width, axis=1), z.width, z.frac)


class Conv2d:
    def __init__(self, s, cin, cout, k, stride=1, pad=0, *, rng, name, seed, frac, width=64, bias=True):
        self.cin, self.cout, self.k, self.stride, self.pad, self.p = cin, cout, k, stride, pad, frac
        fan_in = cin * k * k
        self.W = share_fixed(s, rng.normal(0.0, math.sqrt(2.0 / fan_in), (fan_in, cout)), width, frac,
                             _key(seed, name + ".W"))
        if bias:
            self.b = share_fixed(s, np.zeros(cout), width, frac, _key(seed, name + ".b"))

    def forward(self, s, x):
        n, B, C, H, W = x.values.shape
        self.in_shape = x.values.shape
        self.cols = O.AShare(im2col(x.values, self.k, self.stride, self.pad), x.width, x.frac)
        OH, OW = (H + 2 * self.pad - self.k) // self.stride + 1, (W + 2 * self.pad - self.k) // self.stride + 1
        self.out_hw = (OH, OW)
        z = O.batch_matmul(s, [(self.cols, self.W)])[0]
        if hasattr(self, "b"):
            z = z + _bcast_rows(_lift(self.b, self.p), B * OH * OW)
        z = O.truncate(s, z, self.p)
        v = z.values.reshape(n, B, OH, OW, self.cout).transpose(0, 1, 4, 2, 3)
        return O.AShare(np.ascontiguousarray(v), z.width, z.frac)

    def backward(self, s, dy, need_dx=True):
        n, B, C, H, W = self.in_shape
        OH, OW = self.out_hw
        dz = O.AShare(np.ascontiguousarray(dy.values.transpose(0, 1, 3, 4, 2)).reshape(n, B * OH * OW, self.cout),
                      dy.width, dy.frac)
        pairs = [(_T(self.cols), dz)]
        if need_dx:
            pairs.append((dz, _T(self.W)))
        outs = O.batch_matmul(s, pairs)
        self.gW = outs[0]
        if hasattr(self, "b"):
            self.gb = _colsum(dz)
        if not need_dx:
            return None
        dcols = O.truncate(s, outs[1], self.p)
        return O.AShare(col2im(dcols.values, self.in_shape, self.k, self.stride, self.pad, dcols.width),
                        dcols.width, dcols.frac)

    def step(self, s, shift):
        self.W = self.W - O.truncate(s, self.gW, self.p + shift, out_frac=self.p)
        if hasattr(self, "b"):
            self.b = self.b - O.truncate(s, self.gb, shift, out_frac=self.p)


class AvgPool2d:
    """k x k average pool, stride st (default k): window sum, then / k^2 as a
    truncation by log2(k^2) for power-of-two windows, else scale by the
    public fixed-point 1/k^2 and truncate by p. Backward: the same scaling of
    dy, scattered back over the windows (the sum's adjoint)."""

    def __init__(self, k=2, stride=None):
        self.k = k
        self.st = k if stride is None else stride
        area = k * k
        self.shift = area.bit_length() - 1 if area & (area - 1) == 0 else None

    def _scale(self, s, v: O.AShare) -> O.AShare:
        if self.shift is not None:
            return O.truncate(s, v, self.shift, out_frac=v.frac)
        return O.truncate(s, O.scale_fixed(s, v, 1.0 / (self.k * self.k)), v.frac)

    def _out_hw(self, H, W):
        return (H - self.k) // self.st + 1, (W - self.k) // self.st + 1

    def forward(self, s, x):
        n, B, C, H, W = x.values.shape
        k, st = self.k, self.st
        OH, OW = self._out_hw(H, W)
        self.in_shape = x.values.shape
        acc = np.zeros((n, B, C, OH, OW), U64)
        with np.errstate(over="ignore"):
            for a in range(k):
                for b in range(k):
                    acc += x.values[:, :, :, a:a + st * (OH - 1) + 1:st, b:b + st * (OW - 1) + 1:st]
        return self._scale(s, O.AShare(O.wrap(acc, x.width), x.width, x.frac))

    def backward(self, s, dy, need_dx=True):
        n, B, C, H, W = self.in_shape
        k, st = self.k, self.st
        OH, OW = self._out_hw(H, W)
        d = self._scale(s, dy)
        dx = np.zeros((n, B, C, H, W), U64)
        with np.errstate(over="ignore"):
            for a in range(k):
                for b in range(k):
                    dx[:, :, :, a:a + st * (OH - 1) + 1:st, b:b + st * (OW - 1) + 1:st] += d.values
        return O.AShare(O.wrap(dx, d.width), d.width, d.frac)


class ReLU:
    def forward(self, s, x):
        zero = O.public_ashare(s.n, 0, x.width, x.frac, x.shape)
        self.sign = O.bit2a(s, O.gt(s, x, zero), x.width)
        return O.mul(s, self.sign, x)

    def backward(self, s, dy, need_dx=True):
        return O.mul(s, self.sign, dy)

    def step(self, s, shift):
        pass


class Flatten:
    def forward(self, s, x):
        self.in_shape = x.shape
        return x.reshape((x.shape[0], int(np.prod(x.shape[1:]))))

    def backward(self, s, dy, need_dx=True):
        return dy.reshape(self.in_shape)

    def step(self, s, shift):
        pass


AvgPool2d.step = lambda self, s, shift: None


class Linear:
    def __init__(self, s, fin, fout, *, rng, name, seed, frac, width=64, bias=True):
        self.p = frac
        self.W = share_fixed(s, rng.normal(0.0, math.sqrt(2.0 / fin), (fin, fout)), width, frac,
                             _key(seed, name + ".W"))
        if bias:
            self.b = share_fixed(s, np.zeros(fout), width, frac, _key(seed, name + ".b"))

    def forward(self, s, x):
        self.x = x
        z = O.batch_matmul(s, [(x, self.W)])[0]
        if hasattr(self, "b"):
            z = z + _bcast_rows(_lift(self.b, self.p), x.shape[0])
        return O.truncate(s, z, self.p)

    def backward(self, s, dy, need_dx=True):
        pairs = [(_T(self.x), dy)]
        if need_dx:
            pairs.append((dy, _T(self.W)))
        outs = O.batch_matmul(s, pairs)
        self.gW = outs[0]
        if hasattr(self, "b"):
            self.gb = _colsum(dy)
        return O.truncate(s, outs[1], self.p) if need_dx else None

    def step(self, s, shift):
        self.W = self.W - O.truncate(s, self.gW, self.p + shift, out_frac=self.p)
        if hasattr(self, "b"):
            self.b = self.b - O.truncate(s, self.gb, shift, out_frac=self.p)


class Model:
    def __init__(self, layers):
        self.layers = list(layers)

    def forward(self, s, x):
        for layer in self.layers:
            x = layer.forward(s, x)
        return x

    def train_step(self, s, x, y, lr_shift):
        B = x.shape[0]
        bshift = int(round(math.log2(B)))
        with s.scope("forward"):
            logits = self.forward(s, x)
        with s.scope("loss"):
            dz = O.softmax(s, logits) - y
        with s.scope("backward"):
            g = dz
            for i in range(len(self.layers) - 1, -1, -1):
                g = self.layers[i].backward(s, g, need_dx=i > 0)
        with s.scope("sgd"):
            for layer in self.layers:
                layer.step(s, lr_shift + bshift)
        return logits


def lenet(s, seed=7, frac=23):
    """Paper Table 'LeNet': 430,500 weights, no biases."""
    rng = np.random.default_rng(seed)
    kw = dict(seed=seed, frac=frac, bias=False)
    return Model([Conv2d(s, 1, 20, 5, rng=rng, name="conv1", **kw), AvgPool2d(2), ReLU(),
                  Conv2d(s, 20, 50, 5, rng=rng, name="conv2", **kw), AvgPool2d(2), ReLU(), Flatten(),
                  Linear(s, 800, 500, rng=rng, name="fc1", **kw), ReLU(),
                  Linear(s, 500, 10, rng=rng, name="fc2", **kw)])


def alexnet(s, seed=7, frac=23):
    """Paper Table 'AlexNet', CIFAR-10 3x32x32: 2,552,874
    parameters = bias-free convolutions + fully-connected layers with bias."""
    rng = np.random.default_rng(seed)
    kw = dict(seed=seed, frac=frac)
    return Model([Conv2d(s, 3, 96, 11, 4, 9, rng=rng, name="conv1", bias=False, **kw), AvgPool2d(3, 2), ReLU(),
                  Conv2d(s, 96, 256, 5, 1, 1, rng=rng, name="conv2", bias=False, **kw), AvgPool2d(2, 1), ReLU(),
                  Conv2d(s, 256, 384, 3, 1, 1, rng=rng, name="conv3", bias=False, **kw), ReLU(),
                  Conv2d(s, 384, 256, 3, 1, 1, rng=rng, name="conv4", bias=False, **kw), ReLU(), Flatten(),
                  Linear(s, 256, 256, rng=rng, name="fc1", **kw), ReLU(),
                  Linear(s, 256, 256, rng=rng, name="fc2", **kw), ReLU(),
                  Linear(s, 256, 10, rng=rng, name="fc3", **kw)])


def vgg16m(s, seed=7, frac=26):
    """Paper Table 'VGG16m', CIFAR-10 3x32x32, p = 26:
    bias-free 3x3 convolutions, fully-connected layers with bias."""
    rng = np.random.default_rng(seed)
    kw = dict(seed=seed, frac=frac)
    layers = []
    cin = 3
    for i, (cout, pool) in enumerate([(64, False), (64, True), (128, False), (128, True), (256, False),
                                      (256, True), (512, False), (512, True), (512, True)]):
        layers.append(Conv2d(s, cin, cout, 3, 1, 1, rng=rng, name=f"conv{i + 1}", bias=False, **kw))
        if pool:
            layers.append(AvgPool2d(2))
        layers.append(ReLU())
        cin = cout
    layers += [Flatten(), Linear(s, 512, 256, rng=rng, name="fc1", **kw), ReLU(),
               Linear(s, 256, 256, rng=rng, name="fc2", **kw), ReLU(),
               Linear(s, 256, 10, rng=rng, name="fc3", **kw)]
    return Model(layers)


def simple_mlp(s, seed=7, frac=23):
    rng = np.random.default_rng(seed)
    kw = dict(seed=seed, frac=frac)
    return Model([Linear(s, 784, 128, rng=rng, name="fc1", **kw), ReLU(),
                  Linear(s, 128, 128, rng=rng, name="fc2", **kw), ReLU(),
                  Linear(s, 128, 10, rng=rng, name="fc3", **kw)])
