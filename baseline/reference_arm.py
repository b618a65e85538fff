"""The reference arm: the UNMODIFIED reference package (``baseline/_ref``, pip-installed
from /root/reference/pkg) timed on the host cores.

Installed once with
    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>
(``--no-deps``: matplotlib is not in the image; the reference imports it only
for plotting in ``report.py:16-18``, so a throwaway stub module satisfies the
import). Everything below calls the reference's own public API and code
path - ``PartySession`` per party thread over ``InProcHub``, ``memory_stores``
(its dealer), ``protocols`` / ``nonlinear`` / ``nn`` - nothing of the B200
engine.

The reference has no training code, so the LeNet step is the
composition ``oracle/train_sim.py`` restates (im2col Conv2d, AvgPool2d,
ReLU, Linear, softmax-CE, SGD) written over the reference's per-party
primitives; ``tests/test_reference_arm.py`` pins it bit-exactly to the oracle
(and so to the GPU engine) on every party's logits and weights.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
import tempfile
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
U64 = np.uint64


def available() -> str | None:
    """None when the installed reference imports, else the reason."""
    if not os.path.isdir(os.path.join(REF_DIR, "mpfix")):
        return f"{REF_DIR} is missing (pip install --target baseline/_ref the reference)"
    try:
        load()
    except Exception as e:  # noqa: BLE001
        return f"reference import failed: {e}"
    return None


_MPFIX = None


def load():
    """Import the installed reference (``mpfix``) with a matplotlib stub."""
    global _MPFIX
    if _MPFIX is not None:
        return _MPFIX
    stub = tempfile.mkdtemp(prefix="mplstub_")
    os.makedirs(os.path.join(stub, "matplotlib"))
    with open(os.path.join(stub, "matplotlib", "__init__.py"), "w") as fh:
        fh.write("def use(*a, **k):\n    pass\n")
    with open(os.path.join(stub, "matplotlib", "pyplot.py"), "w") as fh:
        fh.write("def __getattr__(n):\n    return lambda *a, **k: None\n")
    for p in (REF_DIR, stub):
        if p not in sys.path:
            sys.path.insert(0, p)
    import mpfix  # noqa: F401
    import mpfix.nn
    import mpfix.nonlinear
    import mpfix.preprocessing
    import mpfix.protocols
    import mpfix.ring
    import mpfix.session
    import mpfix.sharing
    import mpfix.transport
    _MPFIX = mpfix
    return mpfix


# ---------------------------------------------------------------------------
# harness (tests/helpers.py:17-49 of the reference): dry run, dealer, threads


def deal(fn, n: int, seed: int = 11) -> list[dict]:
    """Dry run of fn on party 0 (NullMesh + DemandCounter), then the
    reference dealer: per-party {key: (count, arrays)}."""
    M = load()
    from mpfix.metrics import CommMetrics
    counter = M.preprocessing.DemandCounter(party=0)
    fn(M.session.PartySession(0, n, M.transport.NullMesh(0, n), counter, metrics=CommMetrics(0, n)))
    stores = M.preprocessing.memory_stores(seed, n, dict(counter.demands))
    return [{k: (st._counts[k], st._arrays[k]) for k in st._counts} for st in stores]


def fresh_stores(dealt: list[dict]):
    """New reference MaterialStores (cursors at 0) over already dealt arrays."""
    M = load()
    stores = []
    for p, per in enumerate(dealt):
        st = M.preprocessing.MaterialStore(p)
        for k, (count, arrays) in per.items():
            st.add_material(k, count, arrays)
        stores.append(st)
    return stores


def run_parties(fn, n: int, seed: int = 11, dealt: list[dict] | None = None):
    """fn(session) -> (result, online_seconds) on one thread per party.
    Returns ([results by party], max online seconds over parties)."""
    M = load()
    from mpfix.metrics import CommMetrics
    stores = fresh_stores(dealt if dealt is not None else deal(fn, n, seed))
    hub = M.transport.InProcHub(n)
    out, errs = {}, {}

    def worker(p):
        try:
            s = M.session.PartySession(p, n, hub.mesh(p), stores[p], metrics=CommMetrics(p, n))
            out[p] = fn(s)
        except BaseException as e:  # noqa: BLE001
            errs[p] = e

    ts = [threading.Thread(target=worker, args=(p,)) for p in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[min(errs)]
    return [out[p][0] for p in range(n)], max(out[p][1] for p in range(n))


def deal_ring(s, enc: np.ndarray, width: int, key):
    """Input sharing of the scenarios / tests (scenarios.py:54-64): parties
    1..n-1 draw Philox(key) elements in order, party 0 holds the difference."""
    M = load()
    # keys are two u64 words (scenarios.py:48-51 passes a uint64 array; a
    # Python list holding a word >= 2^63 would be read differently by numpy)
    rng = np.random.Generator(np.random.Philox(key=np.asarray(key, dtype=np.uint64)))
    draws = [M.ring.random_elems(rng, enc.shape, width) for _ in range(s.n_parties - 1)]
    first = enc
    for d in draws:
        first = M.ring.sub(first, d, width)
    return ([first] + draws)[s.party].copy()


def share_fixed(s, floats, width, frac, key):
    M = load()
    enc = M.ring.encode(np.asarray(floats, np.float64), width, frac)
    return M.sharing.AShare(deal_ring(s, enc, width, key), width, frac)


# ---------------------------------------------------------------------------
# Training over the reference's per-party primitives (= oracle/train_sim.py)


def _key(seed, label):
    tag = hashlib.sha256(f"{seed}:param:{label}".encode()).digest()
    return [int.from_bytes(tag[:8], "little"), int.from_bytes(tag[8:16], "little")]


def _wrap(v, width):
    return load().ring.wrap(v, width)


def _im2col(x, k, stride, pad):
    B, C, H, W = x.shape
    OH, OW = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    xp = np.zeros((B, C, H + 2 * pad, W + 2 * pad), U64)
    xp[:, :, pad:pad + H, pad:pad + W] = x
    out = np.empty((B, OH, OW, C, k, k), U64)
    for kh in range(k):
        for kw in range(k):
            out[:, :, :, :, kh, kw] = xp[:, :, kh:kh + stride * OH:stride, kw:kw + stride * OW:stride].transpose(0, 2, 3, 1)
    return out.reshape(B * OH * OW, C * k * k)


def _col2im(cols, shape, k, stride, pad, width):
    B, C, H, W = shape
    OH, OW = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    c = cols.reshape(B, OH, OW, C, k, k)
    xp = np.zeros((B, C, H + 2 * pad, W + 2 * pad), U64)
    with np.errstate(over="ignore"):
        for kh in range(k):
            for kw in range(k):
                xp[:, :, kh:kh + stride * OH:stride, kw:kw + stride * OW:stride] += c[:, :, :, :, kh, kw].transpose(0, 3, 1, 2)
    return _wrap(xp[:, :, pad:pad + H, pad:pad + W].copy(), width)


def _A(values, like):
    return load().sharing.AShare(np.ascontiguousarray(values), like.width, like.frac)


def _T(x):
    return _A(x.values.swapaxes(-1, -2), x)


def _bias_rows(b, p, rows):
    """bias lifted to 2p and broadcast over the product's rows (train_sim._lift / _bcast_rows)."""
    lifted = b.mul_public(1 << p, frac_delta=p)
    return _A(np.broadcast_to(lifted.values[None, :], (rows, lifted.values.shape[0])), lifted)


def _colsum(z):
    return _A(_wrap(z.values.sum(axis=0, dtype=U64), z.width), z)


class Conv2d:
    def __init__(self, s, cin, cout, k, stride=1, pad=0, *, rng, name, seed, frac, width=64, bias=True):
        self.k, self.stride, self.pad, self.p, self.cout = k, stride, pad, frac, cout
        fan_in = cin * k * k
        self.W = share_fixed(s, rng.normal(0.0, math.sqrt(2.0 / fan_in), (fan_in, cout)), width, frac,
                             _key(seed, name + ".W"))
        self.b = share_fixed(s, np.zeros(cout), width, frac, _key(seed, name + ".b")) if bias else None

    def forward(self, s, x):
        P = load().protocols
        B, C, H, W = x.shape
        self.in_shape = x.shape
        self.cols = _A(_im2col(x.values, self.k, self.stride, self.pad), x)
        OH, OW = (H + 2 * self.pad - self.k) // self.stride + 1, (W + 2 * self.pad - self.k) // self.stride + 1
        self.out_hw = (OH, OW)
        z = P.batch_matmul(s, [(self.cols, self.W)])[0]
        if self.b is not None:
            z = z + _bias_rows(self.b, self.p, B * OH * OW)
        z = P.truncate(s, z, self.p)
        return _A(z.values.reshape(B, OH, OW, self.cout).transpose(0, 3, 1, 2), z)

    def backward(self, s, dy, need_dx=True):
        P = load().protocols
        B, C, H, W = self.in_shape
        OH, OW = self.out_hw
        dz = _A(dy.values.transpose(0, 2, 3, 1).reshape(B * OH * OW, self.cout), dy)
        pairs = [(_T(self.cols), dz)] + ([(dz, _T(self.W))] if need_dx else [])
        outs = P.batch_matmul(s, pairs)
        self.gW = outs[0]
        if self.b is not None:
            self.gb = _colsum(dz)
        if not need_dx:
            return None
        dcols = P.truncate(s, outs[1], self.p)
        return _A(_col2im(dcols.values, self.in_shape, self.k, self.stride, self.pad, dcols.width), dcols)

    def step(self, s, shift):
        P = load().protocols
        self.W = self.W - P.truncate(s, self.gW, self.p + shift, out_frac=self.p)
        if self.b is not None:
            self.b = self.b - P.truncate(s, self.gb, shift, out_frac=self.p)


class AvgPool2d:
    """Window sum, then / k^2: truncation by log2(k^2) for power-of-two
    windows, else public scale + truncation (train_sim.AvgPool2d)."""

    def __init__(self, k=2, stride=None):
        self.k = k
        self.st = k if stride is None else stride
        area = k * k
        self.shift = area.bit_length() - 1 if area & (area - 1) == 0 else None

    def _scale(self, s, v):
        P = load().protocols
        if self.shift is not None:
            return P.truncate(s, v, self.shift, out_frac=v.frac)
        return P.truncate(s, P.scale_fixed(s, v, 1.0 / (self.k * self.k)), v.frac)

    def _out_hw(self, H, W):
        return (H - self.k) // self.st + 1, (W - self.k) // self.st + 1

    def forward(self, s, x):
        B, C, H, W = x.shape
        k, st = self.k, self.st
        OH, OW = self._out_hw(H, W)
        self.in_shape = x.shape
        acc = np.zeros((B, C, OH, OW), U64)
        with np.errstate(over="ignore"):
            for a in range(k):
                for b in range(k):
                    acc += x.values[:, :, a:a + st * (OH - 1) + 1:st, b:b + st * (OW - 1) + 1:st]
        return self._scale(s, _A(_wrap(acc, x.width), x))

    def backward(self, s, dy, need_dx=True):
        B, C, H, W = self.in_shape
        k, st = self.k, self.st
        OH, OW = self._out_hw(H, W)
        d = self._scale(s, dy)
        dx = np.zeros((B, C, H, W), U64)
        with np.errstate(over="ignore"):
            for a in range(k):
                for b in range(k):
                    dx[:, :, a:a + st * (OH - 1) + 1:st, b:b + st * (OW - 1) + 1:st] += d.values
        return _A(_wrap(dx, d.width), d)

    def step(self, s, shift):
        pass


class ReLU:
    def forward(self, s, x):
        M = load()
        zero = M.sharing.public_ashare(0, x.width, x.frac, s.party, x.shape)
        self.sign = M.protocols.bit2a(s, M.protocols.gt(s, x, zero), x.width)
        return M.protocols.mul(s, self.sign, x)

    def backward(self, s, dy, need_dx=True):
        return load().protocols.mul(s, self.sign, dy)

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


class Linear:
    def __init__(self, s, fin, fout, *, rng, name, seed, frac, width=64, bias=True):
        self.p = frac
        self.W = share_fixed(s, rng.normal(0.0, math.sqrt(2.0 / fin), (fin, fout)), width, frac,
                             _key(seed, name + ".W"))
        self.b = share_fixed(s, np.zeros(fout), width, frac, _key(seed, name + ".b")) if bias else None

    def forward(self, s, x):
        P = load().protocols
        self.x = x
        z = P.batch_matmul(s, [(x, self.W)])[0]
        if self.b is not None:
            z = z + _bias_rows(self.b, self.p, x.shape[0])
        return P.truncate(s, z, self.p)

    def backward(self, s, dy, need_dx=True):
        P = load().protocols
        pairs = [(_T(self.x), dy)] + ([(dy, _T(self.W))] if need_dx else [])
        outs = P.batch_matmul(s, pairs)
        self.gW = outs[0]
        if self.b is not None:
            self.gb = _colsum(dy)
        return P.truncate(s, outs[1], self.p) if need_dx else None

    def step(self, s, shift):
        P = load().protocols
        self.W = self.W - P.truncate(s, self.gW, self.p + shift, out_frac=self.p)
        if self.b is not None:
            self.b = self.b - P.truncate(s, self.gb, shift, out_frac=self.p)


class Model:
    def __init__(self, layers):
        self.layers = list(layers)

    def train_step(self, s, x, y, lr_shift):
        M = load()
        bshift = int(round(math.log2(x.shape[0])))
        with s.scope("forward"):
            logits = x
            for layer in self.layers:
                logits = layer.forward(s, logits)
        with s.scope("loss"):
            dz = M.nn.softmax(s, logits) - y
        with s.scope("backward"):
            g = dz
            for i in range(len(self.layers) - 1, -1, -1):
                g = self.layers[i].backward(s, g, need_dx=i > 0)
        with s.scope("sgd"):
            for layer in self.layers:
                layer.step(s, lr_shift + bshift)
        return logits


def lenet(s, seed=7, frac=23) -> Model:
    """PAPER.md:1317-1346 (train_sim.lenet): bias-free."""
    rng = np.random.default_rng(seed)
    kw = dict(seed=seed, frac=frac, bias=False)
    return Model([Conv2d(s, 1, 20, 5, rng=rng, name="conv1", **kw), AvgPool2d(2), ReLU(),
                  Conv2d(s, 20, 50, 5, rng=rng, name="conv2", **kw), AvgPool2d(2), ReLU(), Flatten(),
                  Linear(s, 800, 500, rng=rng, name="fc1", **kw), ReLU(),
                  Linear(s, 500, 10, rng=rng, name="fc2", **kw)])


def alexnet(s, seed=7, frac=23) -> Model:
    """PAPER.md:1348-1389 (train_sim.alexnet)."""
    rng = np.random.default_rng(seed)
    kw = dict(seed=seed, frac=frac)
    return Model([Conv2d(s, 3, 96, 11, 4, 9, rng=rng, name="conv1", bias=False, **kw), AvgPool2d(3, 2), ReLU(),
                  Conv2d(s, 96, 256, 5, 1, 1, rng=rng, name="conv2", bias=False, **kw), AvgPool2d(2, 1), ReLU(),
                  Conv2d(s, 256, 384, 3, 1, 1, rng=rng, name="conv3", bias=False, **kw), ReLU(),
                  Conv2d(s, 384, 256, 3, 1, 1, rng=rng, name="conv4", bias=False, **kw), ReLU(), Flatten(),
                  Linear(s, 256, 256, rng=rng, name="fc1", **kw), ReLU(),
                  Linear(s, 256, 256, rng=rng, name="fc2", **kw), ReLU(),
                  Linear(s, 256, 10, rng=rng, name="fc3", **kw)])


def vgg16m(s, seed=7, frac=26) -> Model:
    """PAPER.md:1391-1458 (train_sim.vgg16m)."""
    rng = np.random.default_rng(seed)
    kw = dict(seed=seed, frac=frac)
    layers, cin = [], 3
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


ARCHS = {"lenet": lenet, "alexnet": alexnet, "vgg16m": vgg16m}


def _train_fn(arch, x, y, keys, lr_shift):
    build = ARCHS[arch]

    def fn(s):
        m = build(s)
        p = m.layers[0].p
        xs = share_fixed(s, x, 64, p, keys[0])
        ys = share_fixed(s, y, 64, p, keys[1])
        t0 = time.perf_counter()
        logits = m.train_step(s, xs, ys, lr_shift)
        return (m, logits), time.perf_counter() - t0
    return fn


def train_step(arch, x, y, n: int, keys, seed: int = 11, lr_shift: int = 5, dealt=None):
    """One secure SGD step of ``arch`` on the reference, one thread per party.
    Returns (per-party (model, logits), online seconds = max over parties)."""
    return run_parties(_train_fn(arch, x, y, keys, lr_shift), n, seed, dealt)


def lenet_step(x, y, n: int, keys, seed: int = 11, lr_shift: int = 5):
    return train_step("lenet", x, y, n, keys, seed, lr_shift)


# ---------------------------------------------------------------------------
# 18.9M Transformer forward (= oracle/transformer_sim.py) and single ops


def _tkey(seed, label):
    tag = hashlib.sha256(f"{seed}:tparam:{label}".encode()).digest()
    return [int.from_bytes(tag[:8], "little"), int.from_bytes(tag[8:16], "little")]


def transformer_forward(x, n: int, layers=6, d=512, heads=8, ffn=2048, frac=14, seed=7, key=(5, 5), mseed=11):
    """Secure inference of the 6-layer encoder on the reference (transformer_sim)."""
    M = load()
    from oracle.transformer_sim import init_weights   # public float weights (plaintext init only)
    Ws = init_weights(layers, d, ffn, heads, seed)
    dh = d // heads

    def fn(s):
        P, NN = M.protocols, M.nn
        W = [{nm: share_fixed(s, w, 64, frac, _tkey(seed, f"{i}.{nm}")) for nm, w in lw.items()}
             for i, lw in enumerate(Ws)]
        h = share_fixed(s, x, 64, frac, list(key))
        t0 = time.perf_counter()
        S = x.shape[0]
        for i in range(layers):
            Wi = W[i]
            with s.scope(f"layer{i}"):
                with s.scope("qkv"):
                    q, k, v = (P.truncate(s, z, frac) for z in
                               P.batch_matmul(s, [(h, Wi["q"]), (h, Wi["k"]), (h, Wi["v"])]))
                split = lambda t: [_A(t.values.reshape(S, heads, dh)[:, j], t) for j in range(heads)]  # noqa: E731
                with s.scope("attention"):
                    a = NN.attention_block(s, list(zip(split(q), split(k), split(v))), optimized=True)
                a = _A(a.values.transpose(1, 0, 2).reshape(S, d), a)
                with s.scope("proj"):
                    h = h + P.truncate(s, P.batch_matmul(s, [(a, Wi["o"])])[0], frac)
                with s.scope("ffn"):
                    f = NN.relu(s, P.truncate(s, P.batch_matmul(s, [(h, Wi["f1"])])[0], frac))
                    h = h + P.truncate(s, P.batch_matmul(s, [(f, Wi["f2"])])[0], frac)
        return h, time.perf_counter() - t0

    return run_parties(fn, n, mseed)


def op_sample(op: str, enc: np.ndarray, n: int, key, frac: int = 23, seed: int = 11):
    """Online reciprocal / exponentiation / logarithm (nonlinear.py:146-267) on the reference."""
    M = load()
    f = {"reciprocal": M.nonlinear.reciprocal, "exp": M.nonlinear.exponentiation,
         "log": M.nonlinear.logarithm}[op]

    def fn(s):
        x = M.sharing.AShare(deal_ring(s, enc, 64, key), 64, frac)
        t0 = time.perf_counter()
        y = f(s, x)
        return y, time.perf_counter() - t0

    return run_parties(fn, n, seed)


def reciprocal_sample(enc: np.ndarray, n: int, key, seed: int = 11):
    return op_sample("reciprocal", enc, n, key, seed=seed)


def matmul_sample(a: np.ndarray, b: np.ndarray, n: int, keys, seed: int = 11):
    """Online Beaver matmul (basic.py:45-79) on the reference."""
    M = load()

    def fn(s):
        x = M.sharing.AShare(deal_ring(s, a, 64, keys[0]), 64, 0)
        y = M.sharing.AShare(deal_ring(s, b, 64, keys[1]), 64, 0)
        t0 = time.perf_counter()
        z = M.protocols.batch_matmul(s, [(x, y)])[0]
        return z, time.perf_counter() - t0

    return run_parties(fn, n, seed)


# ---------------------------------------------------------------------------
# process pool: the batch (or element range) split over host cores


def _pool_task(args):
    kind, payload = args
    if kind == "train":
        arch, x, y, n, keys = payload
        return train_step(arch, x, y, n, keys)[1]
    if kind == "op":
        op, enc, n, key = payload
        return op_sample(op, enc, n, key)[1]
    if kind == "matmul":
        a, b, n, keys = payload
        return matmul_sample(a, b, n, keys)[1]
    if kind == "transformer":
        x, n = payload
        return transformer_forward(x, n)[1]
    if kind == "transformer_layer":     # one of the 6 layers: a bounded latency sample
        x, n = payload
        return transformer_forward(x, n, layers=1)[1]
    raise ValueError(kind)


def parallel_online(tasks: list, procs: int) -> float:
    """Run the tasks on ``procs`` forked processes at once; the slowest
    task's online seconds (all run concurrently) bound the whole sample."""
    import multiprocessing as mp
    load()
    with mp.get_context("fork").Pool(procs) as pool:
        return max(pool.map(_pool_task, tasks, chunksize=1))


def _train_worker(conn, arch, x, y, n, keys, lr_shift):
    fn = _train_fn(arch, x, y, keys, lr_shift)
    dealt = deal(fn, n)
    conn.send("ready")
    while conn.recv() == "step":
        conn.send(run_parties(fn, n, dealt=dealt)[1])
    conn.close()


class TrainWorkers:
    """The batch split over ``procs`` persistent processes (each: one thread
    per party). The dry run and the reference dealer run once per process at
    start-up; every ``step()`` runs the online phase of one SGD step on every
    slice at once (fresh stores over the dealt arrays) and returns the
    slowest slice's online seconds."""

    def __init__(self, arch, x, y, n, keys, procs, lr_shift=5):
        import multiprocessing as mp
        load()
        ctx = mp.get_context("fork")
        bounds = np.linspace(0, len(x), procs + 1).astype(int)
        self.conns, self.procs = [], []
        for i in range(procs):
            a, b = bounds[i], bounds[i + 1]
            if b <= a:
                continue
            mine, theirs = ctx.Pipe()
            pr = ctx.Process(target=_train_worker, args=(theirs, arch, x[a:b], y[a:b], n, keys, lr_shift),
                             daemon=True)
            pr.start()
            self.conns.append(mine)
            self.procs.append(pr)
        for c in self.conns:
            assert c.recv() == "ready"

    def step(self) -> float:
        for c in self.conns:
            c.send("step")
        return max(c.recv() for c in self.conns)

    def close(self):
        for c in self.conns:
            c.send("stop")
        for pr in self.procs:
            pr.join(timeout=30)
