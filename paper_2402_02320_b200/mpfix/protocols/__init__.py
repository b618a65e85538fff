"""``mpfix.protocols`` (protocols/__init__.py:1-30): the reference signatures
over ``mpfix`` handles, each call running the engine's protocol kernels."""

from ... import protocols as _EP
from .._bridge import wrap_op

__all__ = [
    "mul", "matmul", "batch_matmul", "and_gate", "binary_add", "public_add_bits",
    "bit2a", "compose", "decompose", "gt", "add_const", "const_share",
    "truncate", "unsigned_truncate", "scale_fixed", "evaluate_poly",
    "evaluate_square_completed", "lmo", "max_vec",
]

for _nm in __all__:
    globals()[_nm] = wrap_op(getattr(_EP, _nm), _nm)
del _nm
