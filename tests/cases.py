"""Parity cases shared by every engine (reference, CPU oracle, B200 build).

Each case is ``fn(M, s) -> {name: share}`` written against a small engine
namespace ``M`` (see ``tests/engines.py``) so the SAME protocol script runs on
the reference (``/root/reference/pkg``, golden generation only), on the CPU
oracle and on the GPU package. Inputs are dealt exactly like
``/root/reference/pkg/tests/helpers.py:52-78`` (Philox keys [1000+tag, 2] /
[2000+tag, 5], party 0 holds the difference); material comes from the dealer
seeded 11 as in ``helpers.py:17``. The cases mirror the reference's own unit
tests (file:line in each docstring) at fixture-friendly sizes.
"""

from __future__ import annotations

import numpy as np

LOG2E = 1.4426950408889634
LN2 = 0.6931471805599453


def c_mul(M, s):
    """tests/test_basic_protocols.py:14-29"""
    x = M.deal_arith(s, np.arange(400, dtype=np.uint64) * np.uint64(7919), 64, tag=0)
    y = M.deal_arith(s, np.arange(400, dtype=np.uint64) * np.uint64(104729) + np.uint64(5), 64, tag=1)
    return {"z": M.mul(s, x, y)}


def c_mul_w32(M, s):
    """tests/test_basic_protocols.py:32-42"""
    rng = np.random.default_rng(77)
    xs = rng.integers(0, 1 << 32, 256, dtype=np.uint64)
    ys = rng.integers(0, 1 << 32, 256, dtype=np.uint64)
    return {"z": M.mul(s, M.deal_arith(s, xs, 32, tag=0), M.deal_arith(s, ys, 32, tag=1))}


def c_batch_matmul(M, s):
    """tests/test_basic_protocols.py:45-60"""
    rng = np.random.default_rng(9)
    a1 = rng.integers(0, 1 << 63, (5, 7), dtype=np.uint64)
    b1 = rng.integers(0, 1 << 63, (7, 3), dtype=np.uint64)
    a2 = rng.integers(0, 1 << 63, (2, 4), dtype=np.uint64)
    b2 = rng.integers(0, 1 << 63, (4, 6), dtype=np.uint64)
    pairs = [(M.deal_arith(s, a1, 64, tag=0), M.deal_arith(s, b1, 64, tag=1)),
             (M.deal_arith(s, a2, 64, tag=2), M.deal_arith(s, b2, 64, tag=3))]
    o1, o2 = M.batch_matmul(s, pairs)
    return {"o1": o1, "o2": o2}


def c_matmul_square(M, s):
    """tests/test_acceptance.py:41-49 style full-range 20x20 products (3 pairs)."""
    rng = np.random.default_rng(987_001)
    a = rng.integers(0, 1 << 64, (3, 20, 20), dtype=np.uint64)
    b = rng.integers(0, 1 << 64, (3, 20, 20), dtype=np.uint64)
    pairs = [(M.deal_arith(s, a[i], 64, tag=100 + 2 * i), M.deal_arith(s, b[i], 64, tag=101 + 2 * i))
             for i in range(3)]
    return {f"o{i}": o for i, o in enumerate(M.batch_matmul(s, pairs))}


def c_and_xor(M, s):
    """tests/test_basic_protocols.py:63-76"""
    rng = np.random.default_rng(21)
    a = rng.integers(0, 2, 1000, dtype=np.uint8)
    b = rng.integers(0, 2, 1000, dtype=np.uint8)
    x = M.deal_bits(s, a, tag=0)
    y = M.deal_bits(s, b, tag=1)
    return {"and": M.and_gate(s, x, y), "xor": x ^ y}


def c_bit2a(M, s):
    """tests/test_basic_protocols.py:79-87"""
    rng = np.random.default_rng(31)
    bits = rng.integers(0, 2, 500, dtype=np.uint8)
    return {"z": M.bit2a(s, M.deal_bits(s, bits, tag=0), 64)}


def c_decompose_compose(M, s):
    """tests/test_basic_protocols.py:90-101"""
    rng = np.random.default_rng(41)
    xs = rng.integers(0, 1 << 64, 200, dtype=np.uint64)
    x = M.deal_arith(s, xs, 64, tag=0)
    bits = M.decompose(s, x)
    return {"bits": bits, "back": M.compose(s, bits, 64)}


def c_decompose_l8(M, s):
    """tests/test_basic_protocols.py:104-113 (exhaustive l=8)"""
    return {"bits": M.decompose(s, M.deal_arith(s, np.arange(256, dtype=np.uint64), 8, tag=0))}


def c_decompose_w32(M, s):
    rng = np.random.default_rng(43)
    xs = rng.integers(0, 1 << 32, 300, dtype=np.uint64)
    return {"bits": M.decompose(s, M.deal_arith(s, xs, 32, tag=0))}


def c_binary_add_l8(M, s):
    """tests/test_basic_protocols.py:116-129 (l=8, 64x64 sub-grid)"""
    a = np.repeat(np.arange(0, 256, 4, dtype=np.uint64), 64)
    b = np.tile(np.arange(0, 256, 4, dtype=np.uint64) + np.uint64(1), 64)
    x = M.deal_bits(s, M.bits_of(a, 8), tag=0)
    y = M.deal_bits(s, M.bits_of(b, 8), tag=1)
    return {"sum": M.binary_add(s, x, y)}


def c_public_add_bits(M, s):
    """tests/test_basic_protocols.py:132-143"""
    rng = np.random.default_rng(51)
    xs = rng.integers(0, 1 << 16, 128, dtype=np.uint64)
    pub = rng.integers(0, 1 << 16, 128, dtype=np.uint64)
    x = M.deal_bits(s, M.bits_of(xs, 16), tag=0)
    return {"sum": M.public_add_bits(s, M.bits_of(pub, 16), x)}


def c_gt(M, s):
    """tests/test_basic_protocols.py:146-159"""
    rng = np.random.default_rng(61)
    a = rng.integers(-1000, 1000, 600)
    b = rng.integers(-1000, 1000, 600)
    b[:50] = a[:50]
    x = M.deal_arith(s, M.to_ring(a, 64), 64, tag=0)
    y = M.deal_arith(s, M.to_ring(b, 64), 64, tag=1)
    return {"gt": M.gt(s, x, y)}


def c_consts(M, s):
    """tests/test_basic_protocols.py:162-173"""
    c = M.const_share(s, 2.5, 64, 23, shape=(4,))
    x = M.deal_arith(s, M.encode(np.ones(4), 64, 23), 64, frac=23, tag=0)
    return {"c": c, "y": M.add_const(s, x, 1.25)}


def _trunc(f):
    def fn(M, s):
        """tests/test_derived_protocols.py:15-28"""
        rng = np.random.default_rng(100 + f)
        xs = rng.integers(-(1 << 61), 1 << 61, 2000)
        x = M.deal_arith(s, M.to_ring(xs, 64), 64, tag=0)
        return {"z": M.truncate(s, x, f)}
    return fn


def c_unsigned_truncate(M, s):
    """tests/test_derived_protocols.py:31-40"""
    rng = np.random.default_rng(200)
    xs = rng.integers(0, 1 << 62, 1000, dtype=np.uint64)
    return {"z": M.unsigned_truncate(s, M.deal_arith(s, xs, 64, tag=0), 9)}


def c_scale_fixed(M, s):
    """tests/test_derived_protocols.py:43-51"""
    x = M.deal_fixed(s, np.linspace(-30, 30, 101), 64, 23, tag=0)
    y = M.scale_fixed(s, x, LOG2E)
    return {"y": M.truncate(s, y, 23, out_frac=23)}


def c_poly(M, s):
    """tests/test_derived_protocols.py:54-64"""
    x = M.deal_fixed(s, np.linspace(-1.5, 1.5, 61), 64, 23, tag=0)
    return {"y": M.evaluate_poly(s, x, (0.12, -0.8, 0.5, 1.0), 23)}


def c_square_completed(M, s):
    """tests/test_derived_protocols.py:67-79"""
    sq = M.EXP2_SQUARE
    x = M.deal_fixed(s, np.linspace(0.0, 1.0, 33), 64, 23, tag=0)
    return {"y": M.evaluate_square_completed(s, x, sq.lead_shift, sq.t3, sq.t2,
                                             sq.lead * sq.t1, sq.lead * sq.t0, 23)}


def c_lmo_l8(M, s):
    """tests/test_derived_protocols.py:82-90"""
    bits = M.deal_bits(s, M.bits_of(np.arange(256, dtype=np.uint64), 8), tag=0)
    return {"oh": M.lmo(s, bits)}


def c_lmo_after_decompose(M, s):
    """tests/test_derived_protocols.py:93-103"""
    rng = np.random.default_rng(300)
    xs = rng.integers(1, 1 << 50, 128, dtype=np.uint64)
    return {"oh": M.lmo(s, M.decompose(s, M.deal_arith(s, xs, 64, tag=0)))}


def c_max_vec(M, s):
    """tests/test_derived_protocols.py:106-116"""
    rng = np.random.default_rng(400)
    x = M.deal_fixed(s, rng.normal(0, 20, (40, 13)), 64, 23, tag=0)
    return {"m": M.max_vec(s, x)}


def c_reciprocal(M, s):
    """tests/test_nonlinear.py:17-27"""
    xs = np.concatenate([np.logspace(-6, 6, 40, base=2), -np.logspace(-6, 6, 40, base=2)])
    return {"y": M.reciprocal(s, M.deal_fixed(s, xs, 64, 23, tag=0))}


def c_reciprocal_lazy(M, s):
    """tests/test_nonlinear.py:30-45 (newton_iters=1)"""
    x = M.deal_fixed(s, np.logspace(-4, 4, 20, base=2), 64, 23, tag=0)
    return {"y": M.reciprocal(s, x, M.params(newton_iters=1))}


def c_exp_p14(M, s):
    """tests/test_nonlinear.py:48-60"""
    x = M.deal_fixed(s, np.array([-40.0, -16.0, -11.0, -0.5, 0.0, 3.0]), 64, 14, tag=0)
    return {"y": M.exponentiation(s, x)}


def c_exp_p23(M, s):
    """tests/test_nonlinear.py:63-70"""
    return {"y": M.exponentiation(s, M.deal_fixed(s, np.linspace(-6, 6, 49), 64, 23, tag=0))}


def c_attention_exp(M, s):
    """tests/test_nonlinear.py:73-87"""
    xs = np.linspace(-13.5, -0.25, 54)
    a = M.deal_fixed(s, xs, 32, 14, tag=0)
    e = M.deal_fixed(s, xs * LN2, 64, 14, tag=1)
    return {"ya": M.attention_exp(s, a), "ye": M.exponentiation(s, e)}


def c_baseline_exp(M, s):
    """tests/test_nonlinear.py:100-110"""
    x = M.deal_fixed(s, np.array([-4.0, 0.5, 9.0, 12.0]), 64, 16, tag=0)
    return {"y": M.baseline_exp(s, x)}


def c_log(M, s):
    """tests/test_nonlinear.py:113-120"""
    return {"y": M.logarithm(s, M.deal_fixed(s, np.logspace(-7.5, 7.5, 60, base=2), 64, 23, tag=0))}


def c_log_big(M, s):
    """nonlinear.py:230-234 big_input_check path (no reference unit test)."""
    xs = np.array([0.5, 3.0, 1000.0, 2.0 ** 12, 2.0 ** 20, 2.0 ** 30])
    return {"y": M.logarithm(s, M.deal_fixed(s, xs, 64, 16, tag=0), big_input_check=True)}


def c_relu(M, s):
    """tests/test_nn_ops.py:17-24"""
    return {"y": M.relu(s, M.deal_fixed(s, np.linspace(-4, 4, 33), 64, 23, tag=0))}


def c_maxcut(M, s):
    """tests/test_nn_ops.py:27-37"""
    rng = np.random.default_rng(1)
    return {"y": M.maxcut(s, M.deal_fixed(s, rng.normal(0, 5, (5, 11)), 64, 23, tag=0))}


def c_softmax(M, s):
    """tests/test_nn_ops.py:40-49"""
    rng = np.random.default_rng(2)
    return {"y": M.softmax(s, M.deal_fixed(s, rng.normal(0, 6, (12, 64)), 64, 23, tag=0))}


def c_softmax_parts(M, s):
    """tests/test_nn_ops.py:52-62"""
    rng = np.random.default_rng(3)
    e, r = M.softmax_parts(s, M.deal_fixed(s, rng.normal(0, 3, (6, 32)), 64, 23, tag=0))
    return {"e": e, "r": r}


def _attention(optimized):
    def fn(M, s):
        """tests/test_nn_ops.py:79-95"""
        rng = np.random.default_rng(5)
        q = rng.normal(0, 1, (10, 6))
        k = rng.normal(0, 1, (10, 6))
        v = rng.normal(0, 0.5, (10, 6))
        fold = LOG2E / np.sqrt(6)
        head = (M.deal_fixed(s, q, 64, 14, tag=0), M.deal_fixed(s, k * fold, 64, 14, tag=1),
                M.deal_fixed(s, v, 64, 14, tag=2))
        return {"out": M.attention_block(s, [head], optimized=optimized)}
    return fn


def c_attention_heads(M, s):
    """tests/test_nn_ops.py:98-120 (4 heads, both variants)"""
    rng = np.random.default_rng(6)
    heads = []
    for h in range(4):
        q = rng.normal(0, 1, (8, 8))
        k = rng.normal(0, 1, (8, 8))
        v = rng.normal(0, 0.5, (8, 4))
        fold = LOG2E / np.sqrt(8)
        heads.append((M.deal_fixed(s, q, 64, 14, tag=10 + 3 * h),
                      M.deal_fixed(s, k * fold, 64, 14, tag=11 + 3 * h),
                      M.deal_fixed(s, v, 64, 14, tag=12 + 3 * h)))
    return {"naive": M.attention_block(s, heads, optimized=False),
            "opt": M.attention_block(s, heads, optimized=True)}


def c_attention_wide(M, s):
    """tests/test_nn_ops.py:123-141 (cast_width=64)"""
    rng = np.random.default_rng(7)
    q = rng.normal(0, 1, (8, 4))
    k = rng.normal(0, 1, (8, 4))
    v = rng.normal(0, 0.5, (8, 4))
    fold = LOG2E / np.sqrt(4)
    head = (M.deal_fixed(s, q, 64, 14, tag=0), M.deal_fixed(s, k * fold, 64, 14, tag=1),
            M.deal_fixed(s, v, 64, 14, tag=2))
    return {"out": M.attention_block(s, [head], optimized=True, cast_width=64)}


def c_linear(M, s):
    """tests/test_nn_ops.py:144-154"""
    rng = np.random.default_rng(8)
    xs = rng.normal(0, 1, (9, 5))
    layer = M.linear(rng.normal(0, 0.5, (5, 3)), rng.normal(0, 0.1, 3))
    return {"y": M.linear_layer(s, M.deal_fixed(s, xs, 64, 23, tag=0), layer)}


def c_mlp(M, s):
    """tests/test_nn_ops.py:157-169"""
    rng = np.random.default_rng(9)
    xs = rng.normal(0, 1, (20, 16))
    layers = [M.linear(rng.normal(0, 0.25, (16, 12)), rng.normal(0, 0.1, 12)),
              M.linear(rng.normal(0, 0.3, (12, 4)), rng.normal(0, 0.1, 4))]
    return {"y": M.mlp_forward(s, M.deal_fixed(s, xs, 64, 23, tag=0), layers)}


# name -> (fn, parties)
CASES = {
    "mul_n2": (c_mul, 2), "mul_n3": (c_mul, 3), "mul_n4": (c_mul, 4),
    "mul_w32": (c_mul_w32, 2),
    "batch_matmul": (c_batch_matmul, 3),
    "matmul_square": (c_matmul_square, 2),
    "and_xor": (c_and_xor, 4),
    "bit2a": (c_bit2a, 3),
    "decompose_compose": (c_decompose_compose, 2),
    "decompose_l8": (c_decompose_l8, 2),
    "decompose_w32": (c_decompose_w32, 3),
    "binary_add_l8": (c_binary_add_l8, 2),
    "public_add_bits": (c_public_add_bits, 3),
    "gt_n2": (c_gt, 2), "gt_n5": (c_gt, 5),
    "consts": (c_consts, 3),
    "trunc_f1": (_trunc(1), 2), "trunc_f16": (_trunc(16), 2), "trunc_f23": (_trunc(23), 2),
    "unsigned_truncate": (c_unsigned_truncate, 3),
    "scale_fixed": (c_scale_fixed, 2),
    "poly": (c_poly, 2),
    "square_completed": (c_square_completed, 2),
    "lmo_l8": (c_lmo_l8, 2),
    "lmo_after_decompose": (c_lmo_after_decompose, 3),
    "max_vec": (c_max_vec, 2),
    "reciprocal": (c_reciprocal, 2),
    "reciprocal_n3": (c_reciprocal, 3),
    "reciprocal_lazy": (c_reciprocal_lazy, 2),
    "exp_p14": (c_exp_p14, 3),
    "exp_p23": (c_exp_p23, 2),
    "attention_exp": (c_attention_exp, 2),
    "baseline_exp": (c_baseline_exp, 2),
    "log": (c_log, 2),
    "log_big": (c_log_big, 2),
    "relu": (c_relu, 3),
    "maxcut": (c_maxcut, 2),
    "softmax": (c_softmax, 2),
    "softmax_parts": (c_softmax_parts, 2),
    "attention_naive": (_attention(False), 2),
    "attention_opt": (_attention(True), 2),
    "attention_heads": (c_attention_heads, 2),
    "attention_wide": (c_attention_wide, 2),
    "linear": (c_linear, 2),
    "mlp": (c_mlp, 2),
}
