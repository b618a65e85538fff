"""CPU oracle for secure Transformer inference — TEST INFRASTRUCTURE ONLY.

Restates ``paper_2402_02320_b200/transformer.py`` over the oracle primitives
(pinned to the reference); the reference has attention_block but no full
model, so this pins the composition end to end against the GPU build.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

from . import mpc_sim as O


def _key(seed, label):
    tag = hashlib.sha256(f"{seed}:tparam:{label}".encode()).digest()
    return [int.from_bytes(tag[:8], "little"), int.from_bytes(tag[8:16], "little")]


def init_weights(layers, d, ffn, heads, seed=7):
    rng = np.random.default_rng(seed)
    out = []
    scale = 1.0 / math.sqrt(2 * layers)
    dh = d // heads
    for _ in range(layers):
        w = {nm: rng.normal(0.0, scale / math.sqrt(fi), (fi, fo)) for nm, fi, fo in
             (("q", d, d), ("k", d, d), ("v", d, d), ("o", d, d), ("f1", d, ffn), ("f2", ffn, d))}
        w["k"] = w["k"] * (O.LOG2_E / math.sqrt(dh))
        out.append(w)
    return out


def share_fixed(s, floats, width, frac, key):
    enc = O.encode(np.asarray(floats, np.float64), width, frac)
    return O.AShare(O.deal_inputs_arith(enc, s.n, width, key), width, frac)


class Transformer:
    def __init__(self, s, layers=6, d=512, heads=8, ffn=2048, frac=14, width=64, seed=7):
        self.layers, self.d, self.heads, self.p = layers, d, heads, frac
        self.W = [{nm: share_fixed(s, w, width, frac, _key(seed, f"{i}.{nm}")) for nm, w in lw.items()}
                  for i, lw in enumerate(init_weights(layers, d, ffn, heads, seed))]

    def _heads(self, t):
        n, S, _ = t.values.shape
        dh = self.d // self.heads
        v = t.values.reshape(n, S, self.heads, dh).transpose(0, 2, 1, 3)
        return [O.AShare(np.ascontiguousarray(v[:, h]), t.width, t.frac) for h in range(self.heads)]

    def layer(self, s, i, x):
        W, p = self.W[i], self.p
        with s.scope(f"layer{i}"):
            with s.scope("qkv"):
                q, k, v = (O.truncate(s, z, p) for z in O.batch_matmul(s, [(x, W["q"]), (x, W["k"]), (x, W["v"])]))
            with s.scope("attention"):
                a = O.attention_block(s, list(zip(self._heads(q), self._heads(k), self._heads(v))), optimized=True)
            n, H, S, dh = a.values.shape
            a = O.AShare(np.ascontiguousarray(a.values.transpose(0, 2, 1, 3)).reshape(n, S, self.d), a.width, a.frac)
            with s.scope("proj"):
                h = x + O.truncate(s, O.batch_matmul(s, [(a, W["o"])])[0], p)
            with s.scope("ffn"):
                f = O.relu(s, O.truncate(s, O.batch_matmul(s, [(h, W["f1"])])[0], p))
                return h + O.truncate(s, O.batch_matmul(s, [(f, W["f2"])])[0], p)

    def forward(self, s, x):
        for i in range(self.layers):
            x = self.layer(s, i, x)
        return x
