"""``mpfix.nonlinear`` (nonlinear.py:45-356) over the engine: Reciprocal, Exp,
Log, baseline and attention exponentials with the reference's parameters."""

from .. import nonlinear as _EN
from ..nonlinear import DEFAULT_PARAMS, LN2, LOG2_E, ApproxParams, SquareCoeffs  # noqa: F401
from ._bridge import wrap_op

reciprocal = wrap_op(_EN.reciprocal, "reciprocal")
exponentiation = wrap_op(_EN.exponentiation, "exponentiation")
logarithm = wrap_op(_EN.logarithm, "logarithm")
baseline_exp = wrap_op(_EN.baseline_exp, "baseline_exp")
attention_exp = wrap_op(_EN.attention_exp, "attention_exp")

__all__ = ["ApproxParams", "DEFAULT_PARAMS", "SquareCoeffs", "LN2", "LOG2_E", "reciprocal", "exponentiation",
           "logarithm", "baseline_exp", "attention_exp"]
