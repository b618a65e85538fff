"""Golden vectors for the public-value codec and fold_base2 (a35),
produced by running the REFERENCE itself (this container only):

    python tests/golden/make_codec_golden.py

Inputs exercise the edge cases of ring.py:65-121: negatives, exact
multiples and values just below them (floor), ties, the range limits
+-2^(w-1-p), out-of-range magnitudes / inf / NaN (numpy's x86 cast), narrow
widths (8, 31, 32), all sign-boundary words, bit views. fold_base2
(nn.py:58-65) is stored for a layer with and without bias.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from engines import ReferenceEngine  # noqa: E402


def float_inputs():
    rng = np.random.default_rng(45)
    base = [0.0, -0.0, 7.7, -7.7, 0.5, -0.5, 1.0, -1.0, 2.0 ** -23, -(2.0 ** -23), 2.0 ** -24, -(2.0 ** -24),
            1 - 2.0 ** -30, -(1 - 2.0 ** -30), 3.999999999, -3.999999999, 1e-300, -1e-300]
    lims = []
    for w, p in ((64, 23), (64, 14), (32, 14), (64, 0)):
        lim = 2.0 ** (w - 1 - p)
        lims += [lim, -lim, lim * (1 - 2 ** -40), -lim * (1 - 2 ** -40), lim * 2, -lim * 2]
    huge = [2.0 ** 62, 2.0 ** 63, -(2.0 ** 63), 2.0 ** 64, 1e30, -1e30, np.inf, -np.inf, np.nan]
    return np.concatenate([np.array(base + lims + huge), rng.normal(0, 1e3, 200), rng.uniform(-4, 4, 200)])


def main():
    eng = ReferenceEngine()
    ring, nn = eng.ring, eng.mpfix.nn
    xs = float_inputs()
    out = {"x": xs}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for w, p in ((64, 23), (64, 14), (64, 0), (32, 14), (31, 16), (8, 3)):
            out[f"enc_w{w}_p{p}"] = ring.encode(xs, w, p)
    words = np.concatenate([np.arange(0, 300, dtype=np.uint64),
                            np.array([2 ** 63 - 1, 2 ** 63, 2 ** 63 + 1, 2 ** 64 - 1, 2 ** 31 - 1, 2 ** 31,
                                      2 ** 32 - 1, 2 ** 32, 2 ** 30, 2 ** 7, 2 ** 8 - 1], dtype=np.uint64),
                            np.random.default_rng(46).integers(0, 1 << 64, 300, dtype=np.uint64)])
    out["words"] = words
    for w in (64, 32, 31, 8):
        out[f"signed_w{w}"] = ring.to_signed(words, w)
        out[f"bits_w{w}"] = ring.bits_of(words, w)
        out[f"wrap_w{w}"] = ring.wrap(words, w)
        for p in (0, 14, 23):
            if p < w:
                out[f"dec_w{w}_p{p}"] = ring.decode(words, w, p)
    out["cast_64_32"] = ring.cast_down(words, 64, 32)
    out["known_answer"] = np.array([ring.encode(np.array([7.7]), 64, 14)[0]], dtype=np.uint64)
    rng = np.random.default_rng(47)
    W, b = rng.normal(0, 1, (7, 5)), rng.normal(0, 1, 5)
    f1 = nn.fold_base2(nn.LinearLayer(W, b))
    f2 = nn.fold_base2(nn.LinearLayer(W, None))
    out.update({"fold_W": W, "fold_b": b, "fold_W_out": f1.weight, "fold_b_out": f1.bias,
                "fold_W_out_nobias": f2.weight, "fold_nobias_is_none": np.array(f2.bias is None)})
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **out)
    print("wrote", os.path.join(HERE, "codec.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
