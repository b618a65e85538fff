"""Secure training: LeNet / Simple-MLP train steps.

CPU: the B200 training step, run as a dry pass, requests exactly the oracle
restatement's material and records exactly its ledger (same composition and
material order). GPU: one full LeNet train step (forward, softmax-CE,
backward, SGD) is bit-exact against the oracle on every party's logits,
weights and biases; the Simple MLP trained on separable synthetic data
tracks a float64 plaintext twin.
"""

import hashlib
import math

import numpy as np
import pytest
import torch

import oracle as O
from oracle import train_sim as OT


def _key(label):
    tag = hashlib.sha256(f"7:data:{label}".encode()).digest()
    return [int.from_bytes(tag[:8], "little"), int.from_bytes(tag[8:16], "little")]


def _data(B, shape, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, (B,) + shape)
    y = np.eye(10)[rng.integers(0, 10, B)]
    return x, y


def _gpu_lenet_step(s, x, y, B, lr_shift=5, arch="lenet"):
    from paper_2402_02320_b200 import train
    model = getattr(train, arch)(s)
    p = model.layers[0].p
    xs = s.share_fixed(x, 64, p, _key("x"))
    ys = s.share_fixed(y, 64, p, _key("y"))
    logits = model.train_step(s, xs, ys, lr_shift)
    return model, logits


def _oracle_lenet_step(s, x, y, B, lr_shift=5, arch="lenet"):
    model = getattr(OT, arch)(s)
    p = model.layers[0].p
    xs = OT.share_fixed(s, x, 64, p, _key("x"))
    ys = OT.share_fixed(s, y, 64, p, _key("y"))
    logits = model.train_step(s, xs, ys, lr_shift)
    return model, logits


def test_lenet_step_dry_run_matches_oracle_ledger():
    from paper_2402_02320_b200.preprocessing import DemandCounter
    from paper_2402_02320_b200.session import SimSession, demands_by_name
    B, n = 4, 3
    x, y = _data(B, (1, 28, 28))
    c = DemandCounter(tuple(range(n)), n)
    s = SimSession(n, c)
    _gpu_lenet_step(s, x, y, B)
    od = O.Sim(n, O.Demand(n))
    _oracle_lenet_step(od, x, y, B)
    assert demands_by_name(c) == dict(sorted(od.store.demands.items()))
    assert s.metrics.total.as_dict() == od.ledger.total.as_dict()
    assert {k: v.as_dict() for k, v in s.metrics.ledger.items()} == \
        {k: v.as_dict() for k, v in od.ledger.by_scope.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3])
def test_lenet_step_bit_exact_vs_oracle(n):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    B = 4
    x, y = _data(B, (1, 28, 28))
    c = DemandCounter(tuple(range(n)), n)
    _gpu_lenet_step(SimSession(n, c), x, y, B)
    s = SimSession(n, device_store(11, n, c.demands, needs_bits=c.needs_bits))
    gm, gl = _gpu_lenet_step(s, x, y, B)
    torch.cuda.synchronize()
    (om, ol), _ = O.simulate(lambda so: _oracle_lenet_step(so, x, y, B), n, 11)
    assert np.array_equal(gl.values.cpu().numpy().view(np.uint64), ol.values)
    for gl_, ol_ in zip(gm.layers, om.layers):
        for attr in ("W", "b"):
            if hasattr(ol_, attr):
                assert np.array_equal(getattr(gl_, attr).values.cpu().numpy().view(np.uint64),
                                      getattr(ol_, attr).values), (type(ol_).__name__, attr)


@pytest.mark.parametrize("arch", ["alexnet", "vgg16m"])
def test_cifar_nets_dry_run_match_oracle_ledger(arch):
    """configs[2] networks: exact material demand and ledger of one step."""
    from paper_2402_02320_b200.preprocessing import DemandCounter
    from paper_2402_02320_b200.session import SimSession, demands_by_name
    B, n = 2, 2
    x, y = _data(B, (3, 32, 32))
    c = DemandCounter(tuple(range(n)), n)
    s = SimSession(n, c)
    _gpu_lenet_step(s, x, y, B, arch=arch)
    od = O.Sim(n, O.Demand(n))
    _oracle_lenet_step(od, x, y, B, arch=arch)
    assert demands_by_name(c) == dict(sorted(od.store.demands.items()))
    assert s.metrics.total.as_dict() == od.ledger.total.as_dict()


@pytest.mark.gpu
@pytest.mark.parametrize("arch", ["alexnet", "vgg16m"])
def test_cifar_net_step_bit_exact_vs_oracle(arch):
    """configs[2] AlexNet / VGG16m training step (overlapping 3x3/2 and 2x2/1
    average pools, padded strided convolutions) bit-exact vs the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    B, n = 2, 2
    x, y = _data(B, (3, 32, 32))
    c = DemandCounter(tuple(range(n)), n)
    _gpu_lenet_step(SimSession(n, c), x, y, B, arch=arch)
    s = SimSession(n, device_store(11, n, c.demands, needs_bits=c.needs_bits))
    gm, gl = _gpu_lenet_step(s, x, y, B, arch=arch)
    torch.cuda.synchronize()
    (om, ol), _ = O.simulate(lambda so: _oracle_lenet_step(so, x, y, B, arch=arch), n, 11)
    assert np.array_equal(gl.values.cpu().numpy().view(np.uint64), ol.values)
    for gl_, ol_ in zip(gm.layers, om.layers):
        for attr in ("W", "b"):
            if hasattr(ol_, attr):
                assert np.array_equal(getattr(gl_, attr).values.cpu().numpy().view(np.uint64),
                                      getattr(ol_, attr).values), (type(ol_).__name__, attr)


@pytest.mark.gpu
def test_simple_mlp_training_tracks_plaintext():
    """Secure SGD on separable synthetic data follows float64 SGD."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2402_02320_b200 import train
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    n, B, steps, lr_shift = 2, 64, 6, 3
    rng = np.random.default_rng(5)
    centers = rng.normal(0, 1, (10, 784))
    labels = rng.integers(0, 10, B * steps)
    X = centers[labels] + 0.3 * rng.normal(0, 1, (B * steps, 784))
    Y = np.eye(10)[labels]

    def run_secure():
        c = DemandCounter((0, 1), n)
        sd = SimSession(n, c)
        m = train.simple_mlp(sd)
        m.train_step(sd, sd.share_fixed(X[:B], 64, 23, _key("x0")), sd.share_fixed(Y[:B], 64, 23, _key("y0")),
                     lr_shift)
        losses = []
        s = SimSession(n, device_store(11, n, {k: v for k, v in c.demands.items()}, needs_bits=c.needs_bits))
        model = train.simple_mlp(s)
        for t in range(steps):
            st = device_store(100 + t, n, c.demands, needs_bits=c.needs_bits)
            s.store = st
            xs = s.share_fixed(X[t * B:(t + 1) * B], 64, 23, _key(f"x{t}"))
            ys = s.share_fixed(Y[t * B:(t + 1) * B], 64, 23, _key(f"y{t}"))
            logits = s.open_fixed(model.train_step(s, xs, ys, lr_shift))
            p = np.exp(logits - logits.max(1, keepdims=True))
            p /= p.sum(1, keepdims=True)
            losses.append(-np.mean(np.log(p[np.arange(B), labels[t * B:(t + 1) * B]] + 1e-12)))
        return losses

    def run_plain():
        prng = np.random.default_rng(7)
        dims = [(784, 128), (128, 128), (128, 10)]
        Ws = [prng.normal(0, math.sqrt(2 / a), (a, b)) for a, b in dims]
        bs = [np.zeros(b) for _, b in dims]
        losses = []
        lr = 2.0 ** -lr_shift
        for t in range(steps):
            xb, yb = X[t * B:(t + 1) * B], Y[t * B:(t + 1) * B]
            acts = [xb]
            h = xb
            for i, (W, b) in enumerate(zip(Ws, bs)):
                h = h @ W + b
                if i < 2:
                    h = np.maximum(h, 0)
                acts.append(h)
            p = np.exp(h - h.max(1, keepdims=True))
            p /= p.sum(1, keepdims=True)
            losses.append(-np.mean(np.log(p[np.arange(B), labels[t * B:(t + 1) * B]] + 1e-12)))
            g = (p - yb) / B
            for i in (2, 1, 0):
                gW, gb = acts[i].T @ g, g.sum(0)
                if i > 0:
                    g = (g @ Ws[i].T) * (acts[i] > 0)
                Ws[i] -= lr * gW
                bs[i] -= lr * gb
        return losses

    sec, pla = run_secure(), run_plain()
    assert sec[-1] < sec[0] * 0.7
    assert np.allclose(sec, pla, rtol=0.05, atol=0.05), (sec, pla)


@pytest.mark.gpu
def test_graphed_lenet_steps_equal_eager_steps():
    """CUDA-graph replays (in-place re-dealt material) == eager steps, bit for
    bit; building the graph (one eager warm-up step) leaves the weights as they were."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2402_02320_b200 import train
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    n, B, T = 3, 8, 3
    x, y = _data(B, (1, 28, 28))
    c = DemandCounter(tuple(range(n)), n)
    _gpu_lenet_step(SimSession(n, c), x, y, B)

    s1 = SimSession(n, None)
    m1 = train.lenet(s1)
    xs1, ys1 = s1.share_fixed(x, 64, 23, _key("x")), s1.share_fixed(y, 64, 23, _key("y"))
    for t in range(1, T + 1):
        s1.store = device_store(40 + t, n, c.demands, needs_bits=c.needs_bits)
        l1 = m1.train_step(s1, xs1, ys1, 5)

    s2 = SimSession(n, None)
    m2 = train.lenet(s2)
    xs2, ys2 = s2.share_fixed(x, 64, 23, _key("x")), s2.share_fixed(y, 64, 23, _key("y"))
    g = train.GraphedStep(s2, m2, xs2, ys2, 5, c.demands, c.needs_bits, seed0=40)
    for t in range(1, T + 1):
        l2 = g.step(40 + t)
    torch.cuda.synchronize()
    assert torch.equal(l1.values, l2.values)
    for a, b in zip(m1.layers, m2.layers):
        for nm in ("W", "b"):
            if hasattr(a, nm):
                assert torch.equal(getattr(a, nm).values, getattr(b, nm).values), (type(a).__name__, nm)
