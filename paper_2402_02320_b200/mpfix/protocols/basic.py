"""``mpfix.protocols.basic`` names (basic.py:27-239)."""

from . import (add_const, and_gate, batch_matmul, binary_add, bit2a, compose, const_share,  # noqa: F401
               decompose, gt, matmul, mul, public_add_bits)
